#!/bin/bash
# round-2 profiling pass: default bench line, launch list of the bench command, full ncu of the
# cfg5 Schur GEMM launches (all of one factorization), summarised on the box
mkdir -p gpurun_out/r2prof
python bench.py > gpurun_out/r2prof/bench.json 2> gpurun_out/r2prof/bench.err; echo bench rc $?
tail -c 600 gpurun_out/r2prof/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/r2prof/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/r2prof/ncu_launch.log 2>&1; echo ncu-launch rc $?
python tools/ncu_summary.py launches gpurun_out/r2prof/launches_bench.csv > gpurun_out/r2prof/launches_bench.md; head -30 gpurun_out/r2prof/launches_bench.md
gzip -k gpurun_out/r2prof/launches_bench.csv
rm -f gpurun_out/r2prof/launches_bench.csv
ncu --set full --clock-control none --import-source on -k regex:k_gemm_schur -c 80 -o /tmp/full_schur python tools/cfg_once.py cfg5 > gpurun_out/r2prof/ncu_full_schur.log 2>&1; echo ncu-full rc $?
python tools/ncu_summary.py full /tmp/full_schur.ncu-rep k_gemm_schur > gpurun_out/r2prof/ncu_full_k_gemm_schur.json
python -c "import json;print(json.load(open('gpurun_out/r2prof/ncu_full_k_gemm_schur.json'))['summary'])"
ncu --set full --clock-control none --import-source on -k regex:k_gemm_schur -s 24 -c 1 -o gpurun_out/r2prof/schur_one python tools/cfg_once.py cfg5 > /dev/null 2>&1; echo one rc $?
du -sh gpurun_out/r2prof
