# round-2 final records on one B200: GPU tests, cfg3 bench (x2), ncu launch list + one full
# capture of the persistent kernel, cfg2 / cfg4 (swap) / cfg5 (PI sweep) benches, probes
set -x
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/final/gpu_tests_1gpu.log 2>&1; echo tests=$?
for i in 1 2; do python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/final/bench_cfg3.jsonl; done
python bench.py --impl reference --steps 1 --warmup 0 2>/dev/null | tail -1 > gpurun_out/final/bench_cfg3_reference.jsonl
python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/final/bench_cfg2.jsonl
python bench.py --config cfg2 --precision f32 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/final/bench_cfg2.jsonl
for K in 1 8 32; do timeout 900 python bench.py --config cfg5 --K $K --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/final/bench_cfg5_pi_sweep.jsonl; done
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/final/bench_cfg4_swap.jsonl
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --stack-budget 33600000000 --swap-smallest-first 2>/dev/null | tail -1 >> gpurun_out/final/bench_cfg4_swap.jsonl
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --stack-budget 1 2>/dev/null | tail -1 >> gpurun_out/final/bench_cfg4_swap.jsonl
timeout 600 python tools/tc_pipe_probe.py 2>/dev/null | grep "{" > gpurun_out/final/tc_mainloop_probe.jsonl
FLAGS=0,4194304 timeout 300 python tools/fwd_only.py cfg3 5 > gpurun_out/final/fwd_only_phases.log 2>&1
PHASES=1 CHUNKS="8" timeout 600 python tools/dwchunk_ab.py > gpurun_out/final/step_phases.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/cfg3_launches.csv $CMD > gpurun_out/final/ncu_launches.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:cf_driver -s 1 -c 1 -o gpurun_out/final/cfg3_full -f python tools/ncu_one.py --config cfg3 --runs 2 > gpurun_out/final/ncu_full.log 2>&1; echo full=$?
ls -la gpurun_out/final
