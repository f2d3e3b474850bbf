python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); e = d['e2e']; print(round(d['ms_per_step'],2), d['clocks'], '| e2e run', round(e['run_ms_per_step'],2), e['clocks'])"; done
