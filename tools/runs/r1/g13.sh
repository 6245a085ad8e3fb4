mkdir -p gpurun_out/g13
timeout 600 python tools/spike_check.py 16 > gpurun_out/g13/spike.log 2>&1; echo spike rc $?
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g13/bench$i.json 2> gpurun_out/g13/bench$i.err; echo bench rc $?; done
