python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aw_build.log 2>&1
for K in 1 8 32; do
timeout 900 python bench.py --config cfg5 --K $K --steps 3 --warmup 3 2>&1 | tail -1
done
