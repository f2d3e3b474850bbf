python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py -x -q -k "moe or sched" 2>&1 | tail -3
timeout 900 python bench.py --config cfg5 --K 32 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
CF_NO_TC_MATMUL=1 timeout 900 python bench.py --config cfg5 --K 32 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
