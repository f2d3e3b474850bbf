python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do BENCH_DEBUG=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "e2e_ms|^\{" | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('ms', d['ms_per_step'], 'e2e', d['e2e'])
    else: print(l.strip())"; done
