python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aq_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CHUNKS="8" M2ROWS=0,1024 timeout 600 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|phases\|Error"
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-300
