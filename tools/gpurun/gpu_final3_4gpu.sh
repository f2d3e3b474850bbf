mkdir -p gpurun_out/final3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_dp.py tests/test_gpu_control_overhead.py -m gpu -q -rs > gpurun_out/final3/gpu_tests_4gpu.log 2>&1; echo tests=$?
tail -1 gpurun_out/final3/gpu_tests_4gpu.log
timeout 600 python bench.py --gpus 4 --parallel dp --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/final3/bench_cfg3_dp4.jsonl
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/final3/bench_cfg3_pipeline4.jsonl
cut -c1-200 gpurun_out/final3/bench_cfg3_dp4.jsonl gpurun_out/final3/bench_cfg3_pipeline4.jsonl
