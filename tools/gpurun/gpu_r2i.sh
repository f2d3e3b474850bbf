# DXH 256x128 tiles + EW 64-unit tiles: parity, bench, profile
set -x
python -c "import __graft_entry__ as g; g.build(profile=True)" > gpurun_out/r2i_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_swap.py tests/test_gpu_static_unroll.py -x -q -k "bf16 or static" > gpurun_out/r2i_pytest.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_bench.log 2>&1
timeout 600 python tools/profile_run.py --config cfg3 --out gpurun_out/r2i_prof.json > gpurun_out/r2i_prof.log 2>&1
python tools/timeline.py gpurun_out/r2i_prof.npy 30 > gpurun_out/r2i_timeline.txt 2>&1
tail -2 gpurun_out/r2i_pytest.log
cut -c1-300 gpurun_out/r2i_bench.log
head -14 gpurun_out/r2i_timeline.txt
