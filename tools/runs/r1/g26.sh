mkdir -p gpurun_out/g26
timeout 300 python tools/gj_bench.py 256,116 2 > gpurun_out/g26/gj.log 2>&1; echo gj rc $?
