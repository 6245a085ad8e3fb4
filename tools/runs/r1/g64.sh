mkdir -p gpurun_out/g64
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g64/b$i.json 2>gpurun_out/g64/b$i.err; echo b$i rc $?; done
