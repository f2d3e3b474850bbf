# staged coalesced epilogues (fwd + d[x,h]): parity + A/B (flag bit 21 = legacy direct stores)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_swap.py tests/test_gpu_static_unroll.py -x -q -k "bf16 or static" > gpurun_out/r2s_pytest.log 2>&1
echo "pytest exit $?"
FLAGS=0,2097152,0,2097152 timeout 300 python tools/fwd_only.py cfg3 5 > gpurun_out/r2s_fwd.log 2>&1
timeout 300 python tools/driver_cost.py cfg3 0,2097152,0,2097152 > gpurun_out/r2s_ab.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2s_bench.log 2>&1
tail -2 gpurun_out/r2s_pytest.log
cat gpurun_out/r2s_fwd.log
grep flags gpurun_out/r2s_ab.log
cut -c1-200 gpurun_out/r2s_bench.log
