python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_ms'])"; done
python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['ms_per_step'], d['kernel_ms'])"
