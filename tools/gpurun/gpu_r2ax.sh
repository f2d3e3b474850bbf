python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ax_build.log 2>&1
CHUNKS="8" FLAGS=0,256,512,1024,2048 timeout 900 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|Error"
