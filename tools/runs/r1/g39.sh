mkdir -p gpurun_out/g39
FMMLU_TRACE=1 timeout 600 python tools/e2e_spike2.py 25 > gpurun_out/g39/out.log 2> gpurun_out/g39/err.log; echo rc $?
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g39/b$i.json 2>gpurun_out/g39/b$i.err; echo b$i rc $?; done
