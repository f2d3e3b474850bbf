# ncu of the forward-only cfg3 run (current code: staged epilogue, no x-projection split)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v_build.log 2>&1
python tools/fwd_only.py cfg3 2 > gpurun_out/r2v_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cf_driver_kernel -s 1 -c 1 -o gpurun_out/r2v_fwd python tools/fwd_only.py cfg3 2 > gpurun_out/r2v_ncu.log 2>&1
tail -2 gpurun_out/r2v_ncu.log
