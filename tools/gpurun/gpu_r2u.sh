# x-projection ahead of the recurrence: parity + fwd-only A/B (CF_NO_XPROJ) + bench + profile
set -x
python -c "import __graft_entry__ as g; g.build(profile=True)" > gpurun_out/r2u_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_swap.py tests/test_gpu_static_unroll.py -x -q -k "bf16 or static" > gpurun_out/r2u_pytest.log 2>&1
echo "pytest exit $?"
timeout 300 python tools/fwd_only.py cfg3 5 2>&1 | tail -1
CF_NO_XPROJ=1 timeout 300 python tools/fwd_only.py cfg3 5 2>&1 | tail -1
L=1 timeout 300 python tools/fwd_only.py cfg3 5 2>&1 | tail -1
L=1 CF_NO_XPROJ=1 timeout 300 python tools/fwd_only.py cfg3 5 2>&1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_bench.log 2>&1
CF_NO_XPROJ=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_bench_noxp.log 2>&1
timeout 600 python tools/profile_run.py --config cfg3 --out gpurun_out/r2u_prof.json > gpurun_out/r2u_prof.log 2>&1
python tools/timeline.py gpurun_out/r2u_prof.npy 30 > gpurun_out/r2u_timeline.txt 2>&1
tail -2 gpurun_out/r2u_pytest.log
cut -c1-200 gpurun_out/r2u_bench.log gpurun_out/r2u_bench_noxp.log
head -14 gpurun_out/r2u_timeline.txt
