mkdir -p gpurun_out/g15
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g15/bench$i.json 2> gpurun_out/g15/bench$i.err; echo bench rc $?; done
