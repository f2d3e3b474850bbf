python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CF_TEST_KNOBS="2=1" timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "FAILED|passed|failed|info" | tail -4
CHUNKS="8" KNOB2=0,1,0,1 timeout 900 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error" | cut -c1-100
