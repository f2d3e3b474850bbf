# heavy batches: bf16 parity subset + A/B bench (batches on / CF_NO_BATCH) + driver-alone cost
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16" > gpurun_out/r2b_pytest.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench.log 2>&1
CF_NO_BATCH=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_nobatch.log 2>&1
timeout 300 python tools/driver_cost.py cfg3 0,1,0 > gpurun_out/r2b_driver_cost.log 2>&1
CF_NO_BATCH=1 timeout 300 python tools/driver_cost.py cfg3 0,1 > gpurun_out/r2b_driver_cost_nobatch.log 2>&1
tail -3 gpurun_out/r2b_pytest.log
cut -c1-300 gpurun_out/r2b_bench.log gpurun_out/r2b_bench_nobatch.log
cat gpurun_out/r2b_driver_cost.log gpurun_out/r2b_driver_cost_nobatch.log | grep flags
