mkdir -p gpurun_out/g56
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g56/launches.csv python tools/cfg_once.py cfg2 > gpurun_out/g56/ncu.log 2>&1; echo ncu rc $?
python tools/ncu_summary.py launches gpurun_out/g56/launches.csv > gpurun_out/g56/launches.md
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g56/pytest.log 2>&1; echo pytest rc $?
