mkdir -p gpurun_out/g62
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g62/b$i.json 2>gpurun_out/g62/b$i.err; echo b$i rc $?; done
