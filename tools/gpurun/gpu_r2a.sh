set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2a_pytest.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r2a_bench.log 2>&1
echo "bench exit $?"
tail -3 gpurun_out/r2a_pytest.log
