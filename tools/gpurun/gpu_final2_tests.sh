python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/final2
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/final2/gpu_tests_1gpu.log 2>&1; echo tests=$?
tail -1 gpurun_out/final2/gpu_tests_1gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
