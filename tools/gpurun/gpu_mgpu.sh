# N GPUs (N = number visible): multi-GPU parity tests, pipeline + DP benches, f1 ring / barrier
set -x
N=$(python -c "import torch; print(torch.cuda.device_count())")
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mg${N}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_dp.py tests/test_gpu_control_overhead.py -x -q -rs > gpurun_out/mg${N}_pytest.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --gpus $N --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/mg${N}_bench_pipe.log 2>&1
echo "pipe exit $?"
timeout 600 python bench.py --gpus $N --parallel dp --steps 10 --warmup 3 --no-cpu-baseline --watchdog-ms 60000 > gpurun_out/mg${N}_bench_dp.log 2>&1
echo "dp exit $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 tools/control_overhead_mgpu.py --iters 1000 10000 --K 1 32 --barrier > gpurun_out/mg${N}_f1_barrier.jsonl 2> gpurun_out/mg${N}_f1_barrier.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 tools/control_overhead_mgpu.py --iters 1000 10000 --K 1 32 > gpurun_out/mg${N}_f1_ring.jsonl 2> gpurun_out/mg${N}_f1_ring.err
tail -8 gpurun_out/mg${N}_pytest.log
grep -h metric gpurun_out/mg${N}_bench_pipe.log gpurun_out/mg${N}_bench_dp.log | cut -c1-300
cat gpurun_out/mg${N}_f1_barrier.jsonl gpurun_out/mg${N}_f1_ring.jsonl | cut -c1-250
