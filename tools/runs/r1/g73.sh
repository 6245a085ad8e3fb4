# warm cfg5 variance: 5 factorizations on fresh handles in one process, then one traced pair
mkdir -p gpurun_out/g73
timeout 900 python tools/cfg_warm.py cfg5 5 > gpurun_out/g73/c5.json 2> gpurun_out/g73/c5.err; echo c5 rc $?
FMMLU_TRACE=1 timeout 900 python tools/cfg_warm.py cfg5 2 > gpurun_out/g73/c5t.json 2> gpurun_out/g73/c5t.err; echo c5t rc $?
