#!/bin/bash
# pchol_big scratch from the block cache: traced + plain cfg5
mkdir -p gpurun_out/r2_g38
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g38/cfg5t.json 2> gpurun_out/r2_g38/cfg5t.err; grep "allocator host\|L2 host ms" gpurun_out/r2_g38/cfg5t.err | tail -4 | cut -c1-400
timeout 600 python tools/cfg_warm.py cfg5 5 > gpurun_out/r2_g38/cfg5.json 2> /dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_g38/cfg5.json'));print([r['factor_ms'] for r in d['runs']], [r['tree_ms'] for r in d['runs']])"
