N=$(python -c "import torch; print(torch.cuda.device_count())")
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 tools/control_overhead_mgpu.py --iters 1000 10000 --K 1 32 --barrier > gpurun_out/mg${N}_f1_barrier.jsonl 2> gpurun_out/mg${N}_f1_barrier.err
timeout 900 python -m pytest tests/test_gpu_dp.py tests/test_gpu_control_overhead.py -x -q 2>&1 | tail -2
cat gpurun_out/mg${N}_f1_barrier.jsonl
