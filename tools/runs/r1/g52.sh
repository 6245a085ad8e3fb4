mkdir -p gpurun_out/g52
for p in 60 85; do FMMLU_CACHE_PCT=$p FMMLU_TRACE=1 timeout 1200 python tools/cfg_warm.py cfg5 > gpurun_out/g52/c5_$p.json 2> gpurun_out/g52/c5_$p.err; echo p$p rc $?; done
