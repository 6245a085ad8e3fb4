#!/bin/bash
# bench line of the current build + ncu evidence (bounded): launch list of one cfg5 factor+solve,
# full capture of one cfg5 level-6 Schur launch (application replay: no save/restore of 130 GB),
# full captures of every Schur launch of cfg2 (kernel replay)
mkdir -p gpurun_out/r2prof2
python bench.py > gpurun_out/r2prof2/bench.json 2> gpurun_out/r2prof2/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('gpurun_out/r2prof2/bench.json'));print(d['value'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r2prof2/launches_cfg5.csv python tools/cfg_once.py cfg5 > gpurun_out/r2prof2/ncu_launch.log 2>&1; echo ncu-launch rc $?
python tools/ncu_summary.py launches gpurun_out/r2prof2/launches_cfg5.csv > gpurun_out/r2prof2/launches_cfg5.md 2>/dev/null; head -25 gpurun_out/r2prof2/launches_cfg5.md
gzip -f gpurun_out/r2prof2/launches_cfg5.csv
timeout 1200 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_gemm_schur -s 12 -c 1 -o gpurun_out/r2prof2/schur_cfg5_L6 python tools/cfg_once.py cfg5 > gpurun_out/r2prof2/ncu_full_cfg5.log 2>&1; echo ncu-full-cfg5 rc $?
python tools/ncu_summary.py full gpurun_out/r2prof2/schur_cfg5_L6.ncu-rep k_gemm_schur > gpurun_out/r2prof2/ncu_full_k_gemm_schur_cfg5.json 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:k_gemm_schur -c 60 -o /tmp/schur_cfg2 python tools/cfg_once.py cfg2 > gpurun_out/r2prof2/ncu_full_cfg2.log 2>&1; echo ncu-full-cfg2 rc $?
python tools/ncu_summary.py full /tmp/schur_cfg2.ncu-rep k_gemm_schur > gpurun_out/r2prof2/ncu_full_k_gemm_schur_cfg2.json 2>/dev/null
python -c "
import json
for f in ['cfg5','cfg2']:
    try: print(f, json.load(open('gpurun_out/r2prof2/ncu_full_k_gemm_schur_%s.json'%f))['summary'])
    except Exception as e: print(f, e)"
du -sh gpurun_out/r2prof2
