python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2bc_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CHUNKS="8" FLAGS=0,268435456 timeout 900 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error"
timeout 600 python tools/profile_run.py --out gpurun_out/r2bc_prof.json > gpurun_out/r2bc_prof.log 2>&1; echo prof rc=$?
