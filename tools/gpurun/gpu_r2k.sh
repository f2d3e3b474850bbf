# claim-ahead A/B (flag 64 = off), interleaved; parity; bench; driver cost
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1
FLAGS=0,64,0,64,0,64 timeout 300 python tools/fwd_only.py cfg3 5 > gpurun_out/r2k_fwd.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_engine.py -x -q -k "bf16 or tc" > gpurun_out/r2k_pytest.log 2>&1
echo "pytest exit $?"
timeout 300 python tools/driver_cost.py cfg3 0,64,0,64 > gpurun_out/r2k_ab.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_bench.log 2>&1
cat gpurun_out/r2k_fwd.log
tail -2 gpurun_out/r2k_pytest.log
grep flags gpurun_out/r2k_ab.log
cut -c1-300 gpurun_out/r2k_bench.log
