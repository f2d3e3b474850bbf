# round-2 records on 1 GPU: cfg2 latency (bf16 + f32), cfg5 parallel_iterations sweep at
# BASELINE configs[4] (L8 T200 B128, tanh experts), cfg4 long sequence with / without swapping
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rec_build.log 2>&1
for prec in bf16 f32; do
  timeout 300 python bench.py --config cfg2 --precision $prec --steps 20 --warmup 3 --no-cpu-baseline >> gpurun_out/rec_cfg2.jsonl 2>> gpurun_out/rec_err.log
done
for K in 1 8 32; do
  timeout 600 python bench.py --config cfg5 --K $K --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/rec_cfg5.jsonl 2>> gpurun_out/rec_err.log
done
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline >> gpurun_out/rec_cfg4.jsonl 2>> gpurun_out/rec_err.log
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --stack-budget 33600000000 --swap-smallest-first >> gpurun_out/rec_cfg4.jsonl 2>> gpurun_out/rec_err.log
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --stack-budget 1 >> gpurun_out/rec_cfg4.jsonl 2>> gpurun_out/rec_err.log
python - <<'PY'
import json
for f in ["rec_cfg2.jsonl", "rec_cfg5.jsonl", "rec_cfg4.jsonl"]:
    for l in open("gpurun_out/" + f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f, d["config"]["workload"], d["dtype"], "K", d["config"]["parallel_iterations"], "ms %.2f" % d["ms_per_step"],
                  "it/s %.0f" % d["loop_iterations_per_s"], "us/it %.2f" % (d["ms_per_step"] * 1e3 / d["config"]["T"]),
                  "swap", d["stack_swap"]["bytes_d2h"])
PY
tail -5 gpurun_out/rec_err.log
