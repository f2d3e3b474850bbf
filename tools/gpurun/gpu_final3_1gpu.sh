# records after the staging-kernel change: cfg3 bench x2 (full line), launch list, cfg2
mkdir -p gpurun_out/final3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/final3/bench_cfg3.jsonl; done
python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/final3/bench_cfg2.jsonl
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final3/cfg3_launches.csv $CMD > gpurun_out/final3/ncu_launches.log 2>&1; echo launches=$?
ls gpurun_out/final3
