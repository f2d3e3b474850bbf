# round-2 records after the add_dep race fix: GPU tests, smoke, cfg3 bench (x2), cfg2, cfg5 K=32,
# ncu launch list of the cfg3 bench command
set -x
mkdir -p gpurun_out/final2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final2/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/final2/gpu_tests_1gpu.log 2>&1; echo tests=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final2/smoke.log 2>&1; echo smoke=$?
for i in 1 2; do python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/final2/bench_cfg3.jsonl; done
python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/final2/bench_cfg2.jsonl
timeout 900 python bench.py --config cfg5 --K 32 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/final2/bench_cfg5_K32.jsonl
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final2/cfg3_launches.csv $CMD > gpurun_out/final2/ncu_launches.log 2>&1; echo launches=$?
ls -la gpurun_out/final2
