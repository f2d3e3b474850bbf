python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python tools/copy_interference.py 2>&1 | grep "ms per run" | head -6
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); e = d['e2e']; print(round(d['ms_per_step'],2), 'e2e', round(e['value']), 'run', round(e['run_ms_per_step'],2), 'copy', round(e['h2d_ms_per_step'],2), 'launches', d['gpu_launches'])"; done
