set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y_build.log 2>&1
CHUNKS="8 15 12 10" timeout 600 python tools/dwchunk_ab.py 2>&1 | grep dw_chunk
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_swap.py tests/test_gpu_nested.py -x -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 2>&1 | tail -1
