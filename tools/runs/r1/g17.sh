mkdir -p gpurun_out/g17
for m in 0 1; do FMMLU_SCHUR_3M=$m timeout 300 python tools/host_trace.py > gpurun_out/g17/ht$m.log 2>&1; echo m$m rc $?; done
FMMLU_SCHUR_3M=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or residual" > gpurun_out/g17/pytest.log 2>&1; echo pytest rc $?
