mkdir -p gpurun_out/g57
for v in 0 1; do FMMLU_PCHOL_CL8=$v timeout 300 python tools/host_trace.py > gpurun_out/g57/ht$v.log 2>&1; echo h$v rc $?; done
FMMLU_PCHOL_CL8=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or pchol or cfg2_full" > gpurun_out/g57/pytest.log 2>&1; echo pytest rc $?
