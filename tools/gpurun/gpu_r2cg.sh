# A/B of the claim-ahead lead (knob 0: k-blocks before a tile's last MMA; 0 = default 8)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CHUNKS="8" KNOB0=0,4,12,16,24,0 timeout 900 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error" | cut -c1-100
