python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3 4 5 6; do
CHUNKS="8" timeout 300 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error" | tail -1; echo "rc=$?"
done
CF_NO_BATCH_LEVELS=1 CHUNKS="8" timeout 300 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error"
