python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CHUNKS="8" FLAGS=0,256,512,1024,1536 timeout 900 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error"
