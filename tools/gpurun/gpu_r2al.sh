python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2an_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/profile_run.py --out gpurun_out/r2an_prof.json > gpurun_out/r2an_prof.log 2>&1
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-300
CF_NO_ROOT_HINTS=1 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-300
python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-300
