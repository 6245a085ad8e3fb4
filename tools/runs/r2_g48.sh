#!/bin/bash
# ncu --set full of store-GEMM launches around level 6 (Gram / E-F / panel / GJ updates) and of the list kernels
mkdir -p gpurun_out/r2_g48
O=gpurun_out/r2_g48
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_gemm_store$ -s 180 -c 24 -o /tmp/full_store python tools/cfg_warm.py cfg5 1 > $O/ncu_store.log 2>&1; echo ncu store rc $?
python tools/ncu_summary.py full /tmp/full_store.ncu-rep k_gemm_store > $O/full_k_gemm_store.json; python -c "
import json
d=json.load(open('$O/full_k_gemm_store.json'))
for l in d['launches']: print(int(l['grid']), round(l['duration'],3), round(l.get('dmma_pipe_pct') or 0,1), round(l.get('sm_pct') or 0,1), round(((l.get('dram_read') or 0)+(l.get('dram_write') or 0))/1e6,1))
"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_topo_ -c 12 -o /tmp/full_topo python tools/cfg_warm.py cfg5 1 > $O/ncu_topo.log 2>&1; echo ncu topo rc $?
python tools/ncu_summary.py full /tmp/full_topo.ncu-rep k_topo > $O/full_k_topo.json; python -c "
import json
d=json.load(open('$O/full_k_topo.json'))
for l in d['launches']: print(l['kernel'], int(l['grid']), round(l['duration'],3), round(l.get('sm_pct') or 0,1))
"
