python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3 4; do
CHUNKS="8" timeout 300 python tools/dwchunk_ab.py > gpurun_out/r2bt_$i.log 2>&1; echo "run $i rc=$?"; grep dw_chunk gpurun_out/r2bt_$i.log | tail -2
done
