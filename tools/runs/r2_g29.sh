#!/bin/bash
# thresholds: left-looking pivoted Cholesky batch minimum, blocked-GJ batch minimum (class ms on cfg5 / cfg2 / cfg3)
mkdir -p gpurun_out/r2_g29
for ll in 32 64 128; do for gj in 50 100 200; do
  for c in cfg5 cfg2; do
    FMMLU_PCHOL_LL_MIN=$ll FMMLU_GJ_BATCH=$gj timeout 600 python tools/cfg_warm.py $c 3 > gpurun_out/r2_g29/${c}_ll${ll}_gj${gj}.json 2> /dev/null
    python - <<PY
import json
d=json.load(open("gpurun_out/r2_g29/${c}_ll${ll}_gj${gj}.json"))
print("$c ll $ll gj $gj factor", [r["factor_ms"] for r in d["runs"]], "cpqr", d["class_ms"]["cpqr"], "inv", d["class_ms"]["inv"])
PY
  done
done; done
FMMLU_PCHOL_LL_MIN=32 FMMLU_GJ_BATCH=50 timeout 600 python tools/cfg_warm.py cfg3 3 > gpurun_out/r2_g29/cfg3_ll32_gj50.json 2>/dev/null; cut -c1-900 gpurun_out/r2_g29/cfg3_ll32_gj50.json
timeout 600 python tools/cfg_warm.py cfg3 3 > gpurun_out/r2_g29/cfg3_def.json 2>/dev/null; cut -c1-900 gpurun_out/r2_g29/cfg3_def.json
