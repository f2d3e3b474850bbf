#!/bin/bash
# one gpurun call: GPU parity tests, default bench, instance profile of cfg3 (timeline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
timeout 300 python tools/profile_run.py --config cfg3 --out gpurun_out/prof200.json > gpurun_out/prof200.log 2>&1; python tools/chain.py gpurun_out/prof200.npy
echo "prof rc=$?"
python tools/timeline.py gpurun_out/prof200.npy 12
