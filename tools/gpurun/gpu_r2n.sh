# f2 nested frames on the device + regression of the driver changes
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_nested.py -x -q > gpurun_out/r2n_nested.log 2>&1
echo "nested exit $?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_swap.py tests/test_gpu_control_overhead.py tests/test_gpu_static_unroll.py -x -q > gpurun_out/r2n_pytest.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_bench.log 2>&1
tail -30 gpurun_out/r2n_nested.log
tail -3 gpurun_out/r2n_pytest.log
cut -c1-200 gpurun_out/r2n_bench.log
