python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ag_build.log 2>&1
PHASES=1 CHUNKS="8" KNOB0=3,6,10,16 timeout 600 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|phases\|Error"
