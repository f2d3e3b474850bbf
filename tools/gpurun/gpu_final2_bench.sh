# the round-end bench commands on the final bench.py: default N=1, N=2 (torchrun), reference arm
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py 2>/dev/null | tail -1 | cut -c1-250
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 2>/dev/null | tail -1 | cut -c1-250
python bench.py --impl reference --steps 1 --warmup 3 2>/dev/null | tail -1 | cut -c1-250
