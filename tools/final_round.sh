#!/bin/bash
# end-of-round measurement set (1 GPU): bench, ncu launch list + full capture, instance
# profiles, cfg5 parallel_iterations sweep, cfg4 with / without swapping
mkdir -p gpurun_out
bash tools/gpu_profile_session.sh > /dev/null 2>&1; echo profile_session=$?
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python tools/profile_run.py --out gpurun_out/pt.json > /dev/null 2>&1; echo prof=$?
python tools/profile_run.py --no-tiles --out gpurun_out/pnt.json > /dev/null 2>&1; echo prof_nt=$?
for K in 1 8 32; do
  python bench.py --config cfg5 --K $K --no-cpu-baseline --steps 3 > gpurun_out/r_cfg5_K$K.log 2>&1; echo cfg5 K=$K rc=$?
done
python bench.py --config cfg4 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/r_cfg4.log 2>&1; echo cfg4 rc=$?
python bench.py --config cfg4 --no-cpu-baseline --steps 2 --warmup 3 --stack-budget 33600000000 --swap-smallest-first > gpurun_out/r_cfg4_swap_ch.log 2>&1; echo cfg4 swap c,h rc=$?
python bench.py --config cfg4 --no-cpu-baseline --steps 2 --warmup 3 --stack-budget 1 > gpurun_out/r_cfg4_swap_all.log 2>&1; echo cfg4 swap all rc=$?
for f in gpurun_out/bench_full.log gpurun_out/r_*.log; do echo "$f: $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'ms', round(d['roofline']['frac'],3), d['config'].get('parallel_iterations'), d.get('stack_swap',{}).get('bytes_d2h'))" 2>&1 | tail -1)"; done
