#!/bin/bash
# TMA-staged (cp.async.bulk + mbarrier) panel loads in k_gj_panel and column loads in k_pchol_ll: parity + timing
mkdir -p gpurun_out/r2_g34
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "parity_vs_oracle or single_leaf or tight" > gpurun_out/r2_g34/quick.log 2>&1; echo "quick rc=$?"; tail -3 gpurun_out/r2_g34/quick.log
timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g34/cfg5.json 2> gpurun_out/r2_g34/cfg5.err; echo cfg5 rc $?; cut -c1-1100 gpurun_out/r2_g34/cfg5.json; tail -2 gpurun_out/r2_g34/cfg5.err | cut -c1-300
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r2_g34/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_g34/tests.log; grep -E "^FAILED|^ERROR" gpurun_out/r2_g34/tests.log | head -20
timeout 600 python tools/cfg_warm.py cfg2 3 > gpurun_out/r2_g34/cfg2.json 2> /dev/null; cut -c1-700 gpurun_out/r2_g34/cfg2.json
