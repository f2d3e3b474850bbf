# 2 GPUs: pipeline / barrier / DP tests + pipeline and DP benches + f1 barrier numbers
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1
nvidia-smi topo -m > gpurun_out/r2f_topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_dp.py tests/test_gpu_control_overhead.py -x -q -rs > gpurun_out/r2f_pytest.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_pipe2.log 2>&1
timeout 600 python bench.py --gpus 2 --parallel dp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_dp2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/control_overhead_mgpu.py --iters 1000 10000 --K 1 32 --barrier > gpurun_out/r2f_f1_barrier2.jsonl 2> gpurun_out/r2f_f1_barrier2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 tools/control_overhead_mgpu.py --iters 1000 10000 --K 1 32 > gpurun_out/r2f_f1_ring2.jsonl 2> gpurun_out/r2f_f1_ring2.err
tail -8 gpurun_out/r2f_pytest.log
grep -h metric gpurun_out/r2f_bench_pipe2.log gpurun_out/r2f_bench_dp2.log | cut -c1-400
cat gpurun_out/r2f_f1_barrier2.jsonl gpurun_out/r2f_f1_ring2.jsonl
