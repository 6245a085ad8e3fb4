mkdir -p gpurun_out/g30
nproc > gpurun_out/g30/nproc.txt
for i in 1 2 3; do
FMMLU_BLOCKING_SYNC=1 timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g30/block$i.json 2>/dev/null; echo b$i rc $?
timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g30/spin$i.json 2>/dev/null; echo s$i rc $?
done
