mkdir -p gpurun_out/g9
for cfg in "4 256" "1000 256" "1000 128" "8 128" "16 64" "1000 64"; do
set -- $cfg
FMMLU_GRAM_CPS=$1 FMMLU_GRAM_MINCH=$2 timeout 300 python tools/host_trace.py > gpurun_out/g9/ht_$1_$2.log 2>&1; echo $cfg rc $?
done
