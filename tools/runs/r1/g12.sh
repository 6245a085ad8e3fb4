mkdir -p gpurun_out/g12
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g12/bench.json 2> gpurun_out/g12/bench.err; echo bench rc $?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/g12/pytest.log 2>&1; echo pytest rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g12/launches.csv python tools/cfg_once.py cfg2 > gpurun_out/g12/ncu.log 2>&1; echo ncu rc $?
python tools/ncu_summary.py launches gpurun_out/g12/launches.csv > gpurun_out/g12/launches.md
