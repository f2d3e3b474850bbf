python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ae_build.log 2>&1
for ch in 8 2 4 12 16 8; do
CHUNKS="$ch" FLAGS=0 timeout 300 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|phases\|Error\|error" | tail -3
done
