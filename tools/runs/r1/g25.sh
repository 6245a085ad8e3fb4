mkdir -p gpurun_out/g25
timeout 600 ncu --set full --import-source on -k regex:k_gj_blk -c 1 -o gpurun_out/g25/gjblk python tools/gj_bench.py 256 2 > gpurun_out/g25/ncu.log 2>&1; echo ncu rc $?
