python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "moe" 2>&1 | tail -3
CF_NO_TC_MATMUL=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "moe_tensor" 2>&1 | tail -2
