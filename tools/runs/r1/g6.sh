mkdir -p gpurun_out/g6
for m in 0 1 2 3; do
FMMLU_GJ_PANEL=$m timeout 300 python tools/host_trace.py > gpurun_out/g6/panel$m.log 2>&1; echo m$m rc $?
done
