set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1
timeout 600 python tools/dwchunk_ab.py 2>&1 | grep -v "^$" | tail -20
