mkdir -p gpurun_out/g4
timeout 300 python tools/gj_bench.py 64,116,205,256,384 2,8 > gpurun_out/g4/gj.log 2>&1; echo gj rc $?
FMMLU_GJ_TIMING=1 timeout 300 python tools/gj_bench.py 116,256 2 > gpurun_out/g4/gj_timing.log 2>&1; echo gjt rc $?
FMMLU_PCHOL_TIMING=1 timeout 300 python tools/cfg_once.py cfg2 > gpurun_out/g4/pchol_timing.log 2>&1; echo pct rc $?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g4/bench.json 2> gpurun_out/g4/bench.err; echo bench rc $?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g4/pytest.log 2>&1; echo pytest rc $?
