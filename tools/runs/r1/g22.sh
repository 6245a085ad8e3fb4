mkdir -p gpurun_out/g22
timeout 900 python tools/cfg4_bench.py > gpurun_out/g22/cfg4.log 2>&1; echo cfg4 rc $?
timeout 900 python tools/cfg_check.py cfg3 > gpurun_out/g22/cfg3.log 2>&1; echo cfg3 rc $?
timeout 1500 python tools/cfg_check.py cfg5 > gpurun_out/g22/cfg5.log 2>&1; echo cfg5 rc $?
timeout 900 python tools/rcs_bench.py cfg5 1000 > gpurun_out/g22/rcs_cfg5.json 2> gpurun_out/g22/rcs_cfg5.err; echo rcs5 rc $?
