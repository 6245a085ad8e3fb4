mkdir -p gpurun_out/g14
SMI=1 timeout 600 python tools/e2e_spike.py 25 > gpurun_out/g14/e2e_smi.log 2>&1; echo e2e rc $?
