set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2o_build.log 2>&1
for args in "1 1 1" "1 2 1" "2 1,1 1" "2 1,1 32" "5 2,2,2,2,2 1"; do
  timeout 60 python tools/nested_debug.py $args 2>&1 | tail -1
  CF_NO_WAVES=1 timeout 60 python tools/nested_debug.py $args 2>&1 | tail -1
  CF_NO_LEVEL_ORDER=1 timeout 60 python tools/nested_debug.py $args 2>&1 | tail -1
done
