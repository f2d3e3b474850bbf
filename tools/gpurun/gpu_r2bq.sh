python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3 4 5 6 7 8; do
CHUNKS="8" timeout 300 python tools/dwchunk_ab.py > gpurun_out/r2bq_$i.log 2>&1; echo "run $i rc=$?"; grep dw_chunk gpurun_out/r2bq_$i.log | tail -1
done
CF_NO_BATCH_LEVELS=1 CHUNKS="8" timeout 300 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error"
