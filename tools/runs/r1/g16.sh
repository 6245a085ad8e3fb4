mkdir -p gpurun_out/g16
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/g16/pytest.log 2>&1; echo pytest rc $?
timeout 600 python tools/e2e_spike.py 8 > gpurun_out/g16/e2e.log 2>&1; echo e2e rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g16/launches.csv python tools/cfg_once.py cfg2 > gpurun_out/g16/ncu.log 2>&1; echo ncu rc $?
python tools/ncu_summary.py launches gpurun_out/g16/launches.csv > gpurun_out/g16/launches.md
