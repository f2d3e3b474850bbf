# L2 prefetch ahead of the fwd tile's smem ring: A/B distances on the forward-only run, parity, bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1
FLAGS=0,983040,131072,524288,0,983040 timeout 300 python tools/fwd_only.py cfg3 5 > gpurun_out/r2j_fwd.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16" > gpurun_out/r2j_pytest.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_bench.log 2>&1
cat gpurun_out/r2j_fwd.log
tail -2 gpurun_out/r2j_pytest.log
cut -c1-300 gpurun_out/r2j_bench.log
