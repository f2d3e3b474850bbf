# round-end rehearsal on a fresh box: build, GPU suite x3 (flakiness), smoke, default bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3; do timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1; done
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>/dev/null | tail -1 | cut -c1-300
