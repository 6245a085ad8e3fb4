mkdir -p gpurun_out/g24
timeout 300 python tools/gj_bench.py 64,100,116,128,205,256,384 2,8 > gpurun_out/g24/gj.log 2>&1; echo gj rc $?
FMMLU_GJ_BLK=0 timeout 300 python tools/gj_bench.py 116,256 2 > gpurun_out/g24/gj_old.log 2>&1; echo gjo rc $?
timeout 300 python tools/host_trace.py > gpurun_out/g24/host_trace.log 2>&1; echo ht rc $?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/g24/pytest.log 2>&1; echo pytest rc $?
