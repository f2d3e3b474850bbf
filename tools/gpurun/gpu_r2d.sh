# fused waves with helper-evaluated contexts + EW unroll 4: parity, bench, driver cost, fwd-only ncu
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_swap.py tests/test_gpu_control_overhead.py -x -q > gpurun_out/r2d_pytest.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench.log 2>&1
timeout 300 python tools/driver_cost.py cfg3 0,1 > gpurun_out/r2d_driver_cost.log 2>&1
python tools/fwd_only.py cfg3 2 > gpurun_out/r2d_fwd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cf_driver_kernel -s 1 -c 1 -o gpurun_out/r2d_fwd python tools/fwd_only.py cfg3 2 > gpurun_out/r2d_ncu.log 2>&1
tail -3 gpurun_out/r2d_pytest.log
cut -c1-300 gpurun_out/r2d_bench.log
grep flags gpurun_out/r2d_driver_cost.log
cat gpurun_out/r2d_fwd_plain.log
tail -3 gpurun_out/r2d_ncu.log
