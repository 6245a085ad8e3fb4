mkdir -p gpurun_out/g46
for c in 16 8 4; do FMMLU_ROOT_CL=$c timeout 300 python tools/host_trace.py > gpurun_out/g46/ht$c.log 2>&1; echo h$c rc $?; done
FMMLU_ROOT_CL=8 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or tight or single_leaf or cfg2_full" > gpurun_out/g46/pytest.log 2>&1; echo pytest rc $?
