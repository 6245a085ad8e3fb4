mkdir -p gpurun_out/g48
for c in cfg1 cfg3 cfg5; do timeout 1200 python tools/cfg_warm.py $c > gpurun_out/g48/$c.json 2> gpurun_out/g48/$c.err; echo $c rc $?; done
