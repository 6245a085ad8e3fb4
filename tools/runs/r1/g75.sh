# HEAD confirmation: smoke() and the default bench line
mkdir -p gpurun_out/g75
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g75/smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/g75/bench.json 2> gpurun_out/g75/bench.err; echo bench rc $?
