mkdir -p gpurun_out/g36
for m in 0 1; do FMMLU_ROOT_COOP=$m timeout 300 python tools/host_trace.py > gpurun_out/g36/ht$m.log 2>&1; echo m$m rc $?; done
FMMLU_ROOT_COOP=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or tight" > gpurun_out/g36/pytest.log 2>&1; echo pytest rc $?
