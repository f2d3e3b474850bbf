# fwd epilogue prefetch + EW ILP: bf16 parity + bench + instance profile
set -x
python -c "import __graft_entry__ as g; g.build(profile=True)" > gpurun_out/r2c_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16" > gpurun_out/r2c_pytest.log 2>&1
echo "pytest exit $?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench.log 2>&1
timeout 300 python tools/driver_cost.py cfg3 0,1 > gpurun_out/r2c_driver_cost.log 2>&1
timeout 600 python tools/profile_run.py --config cfg3 --out gpurun_out/r2c_prof.json > gpurun_out/r2c_prof.log 2>&1
python tools/timeline.py gpurun_out/r2c_prof.npy 30 > gpurun_out/r2c_timeline.txt 2>&1
python tools/chain.py gpurun_out/r2c_prof.npy 8 > gpurun_out/r2c_chain.txt 2>&1
tail -3 gpurun_out/r2c_pytest.log
cut -c1-300 gpurun_out/r2c_bench.log
grep flags gpurun_out/r2c_driver_cost.log
cat gpurun_out/r2c_chain.txt
head -12 gpurun_out/r2c_timeline.txt
