mkdir -p gpurun_out/g3
timeout 300 python tools/gj_bench.py 64,116,205,256,384 2,8,32 > gpurun_out/g3/gj.log 2>&1; echo gj rc $?
FMMLU_GJ_TIMING=1 timeout 300 python tools/gj_bench.py 116,256 2,32 > gpurun_out/g3/gj_timing.log 2>&1; echo gjt rc $?
