# epilogue unroll fix + L2 evict-last on weights + static unroll (f4)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_static_unroll.py -x -q -k "bf16 or static" > gpurun_out/r2e_pytest.log 2>&1
echo "pytest exit $?"
FLAGS=0,32,0,32 timeout 300 python tools/fwd_only.py cfg3 5 > gpurun_out/r2e_fwd.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_bench.log 2>&1
timeout 900 python tools/static_vs_dynamic.py > gpurun_out/r2e_static.jsonl 2>&1
tail -3 gpurun_out/r2e_pytest.log
cat gpurun_out/r2e_fwd.log
cut -c1-300 gpurun_out/r2e_bench.log
cat gpurun_out/r2e_static.jsonl | tail -12
