mkdir -p gpurun_out/g69
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g69/pytest.log 2>&1; echo pytest rc $?
timeout 300 python tools/host_trace.py > gpurun_out/g69/ht.log 2>&1; echo ht rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g69/launches.csv python tools/cfg_once.py cfg2 > gpurun_out/g69/ncu.log 2>&1; echo ncu rc $?
python tools/ncu_summary.py launches gpurun_out/g69/launches.csv > gpurun_out/g69/launches.md
