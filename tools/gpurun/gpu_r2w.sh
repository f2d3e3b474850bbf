set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w_build.log 2>&1
timeout 600 python tools/roles_ab.py 2>&1 | grep low_first
