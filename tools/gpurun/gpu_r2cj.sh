python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in "" nocopy oneset "" nocopy oneset; do BENCH_E2E_AB=$m python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); e = d['e2e']; print('$m', round(d['ms_per_step'],2), 'run', round(e['run_ms_per_step'],2), 'copy', round(e['h2d_ms_per_step'],2))" ; done
