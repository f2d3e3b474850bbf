set -x
python -c "import __graft_entry__ as g; g.build(profile=True)" > gpurun_out/r2m_build.log 2>&1
FLAGS=0,1048576,0,1048576 timeout 300 python tools/fwd_only.py cfg3 5 > gpurun_out/r2m_fwd.log 2>&1
cat gpurun_out/r2m_fwd.log
