#!/bin/bash
# the separate-ID tests incl. the cross section
mkdir -p gpurun_out/r2_g47
timeout 1200 python -m pytest tests/test_gpu_separate.py -q -m gpu > gpurun_out/r2_g47/sep.log 2>&1; echo "sep rc=$?"; tail -4 gpurun_out/r2_g47/sep.log; grep -E "^E  |^FAILED" gpurun_out/r2_g47/sep.log | head -10 | cut -c1-250
