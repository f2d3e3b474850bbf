set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1
for B in 256 512 1024; do B=$B timeout 300 python tools/fwd_only.py cfg3 3 2>&1 | tail -1; done
for L in 1 2 4; do L=$L timeout 300 python tools/fwd_only.py cfg3 3 2>&1 | tail -1; done
