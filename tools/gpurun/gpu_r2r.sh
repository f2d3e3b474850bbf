set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1
timeout 120 python tools/nested_debug2.py 1,3,2,0,3 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_nested.py -x -q > gpurun_out/r2r_nested.log 2>&1
echo "nested exit $?"
tail -3 gpurun_out/r2r_nested.log
