# round-1 closing pass: warm factorizations of cfg1/cfg3/cfg5 with the final code, cross section, torchrun launcher, GPU tests
mkdir -p gpurun_out/g72
timeout 1200 python tools/cfg_warm.py cfg5 > gpurun_out/g72/c5.json 2> gpurun_out/g72/c5.err; echo c5 rc $?
timeout 600 python tools/cfg_warm.py cfg3 > gpurun_out/g72/c3.json 2> gpurun_out/g72/c3.err; echo c3 rc $?
timeout 600 python tools/cfg_warm.py cfg1 > gpurun_out/g72/c1.json 2> gpurun_out/g72/c1.err; echo c1 rc $?
timeout 600 python tools/rcs_bench.py cfg2 1000 > gpurun_out/g72/rcs_cfg2.json 2> gpurun_out/g72/rcs_cfg2.err; echo rcs rc $?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g72/trun.json 2> gpurun_out/g72/trun.err; echo trun rc $?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g72/pytest.log 2>&1; echo pytest rc $?
