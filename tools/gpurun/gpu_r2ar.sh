python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ar_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-300
python bench.py --config cfg2 --steps 20 --warmup 3 2>&1 | tail -1 | cut -c1-400
