python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py tests/test_gpu_swap.py -x -q 2>&1 | tail -2
PHASES=1 CHUNKS="8" FLAGS=0,8388608 timeout 900 python tools/dwchunk_ab.py 2>&1 | grep "dw_chunk\|phases\|Error"
