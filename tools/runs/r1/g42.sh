mkdir -p gpurun_out/g42
for c in 1 2 4 8; do FMMLU_GJ_PUSH_CL=$c timeout 300 python tools/gj_bench.py 100,128,205,256 2,8 > gpurun_out/g42/gj_$c.log 2>&1; echo c$c rc $?; done
for c in 1 2 8; do FMMLU_GJ_PUSH_CL=$c timeout 300 python tools/host_trace.py > gpurun_out/g42/ht_$c.log 2>&1; echo h$c rc $?; done
