python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2af_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
PHASES=1 CHUNKS="8" FLAGS=0 timeout 300 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|phases\|Error"
