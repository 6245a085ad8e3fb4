mkdir -p gpurun_out/g21
timeout 900 python tools/rcs_bench.py cfg2 1000 > gpurun_out/g21/rcs_cfg2.json 2> gpurun_out/g21/rcs_cfg2.err; echo rcs rc $?
