set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1
timeout 300 python tools/tc_pipe_probe.py > gpurun_out/r2l_probe.jsonl 2>&1
cat gpurun_out/r2l_probe.jsonl | cut -c1-300
