#!/bin/bash
# flakiness check: the full GPU suite three times back to back
mkdir -p gpurun_out/r2_g49
for i in 1 2 3; do
  timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_g49/tests$i.log 2>&1; echo "tests $i rc=$?"; tail -2 gpurun_out/r2_g49/tests$i.log | cut -c1-200; grep -E "^FAILED|^ERROR" gpurun_out/r2_g49/tests$i.log | head -5
done
