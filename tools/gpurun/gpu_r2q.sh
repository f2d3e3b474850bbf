set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2q_build.log 2>&1
timeout 120 python tools/nested_debug2.py 1,3,2,0,3 2>&1 | tail -6
timeout 120 python tools/nested_debug2.py 3,3 2>&1 | tail -6
timeout 120 python tools/nested_debug2.py 3 2>&1 | tail -6
