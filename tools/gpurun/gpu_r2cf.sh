# A/B of the driver's completion-poll period (debug flag bits 8-15, x1000 cycles; 0 = 12000)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CHUNKS="8" FLAGS=0,768,1536,3072,6144,0 timeout 900 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error" | cut -c1-100
