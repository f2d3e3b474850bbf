set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2p_build.log 2>&1
for args in "2 1,1 1" "2 1,2 1" "2 2,1 1" "3 1,1,1 1"; do
  CF_NO_WAVES=1 timeout 60 python tools/nested_debug.py $args 2>&1 | tail -1
done
