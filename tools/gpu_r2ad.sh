set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ad_build.log 2>&1
timeout 300 python tools/one_run.py cfg3 3
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:cf_driver -s 2 -c 1 -o gpurun_out/r2ad_cfg3 -f python tools/one_run.py cfg3 3 > gpurun_out/r2ad_ncu.log 2>&1
tail -3 gpurun_out/r2ad_ncu.log
