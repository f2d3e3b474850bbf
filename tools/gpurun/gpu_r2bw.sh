python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3 4 5 6; do
timeout 900 python -m pytest tests/test_gpu_driver_modes.py tests/test_gpu_sched.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
done
