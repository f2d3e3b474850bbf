set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2z_build.log 2>&1
PHASES=1 CHUNKS="8 12 16" timeout 600 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|phases"
FLAGS=0,4194304 timeout 300 python tools/fwd_only.py cfg3 5 2>&1 | grep -v "^$" | tail -6
L=1 FLAGS=0,4194304 timeout 300 python tools/fwd_only.py cfg3 5 2>&1 | grep -v "^$" | tail -6
