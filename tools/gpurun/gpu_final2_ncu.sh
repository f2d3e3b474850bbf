# ncu --set full of one cfg3 launch on the final tree (after the add_dep race fix)
mkdir -p gpurun_out/final2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:cf_driver -s 1 -c 1 -o gpurun_out/final2/cfg3_full -f python tools/ncu_one.py --config cfg3 --runs 2 > gpurun_out/final2/ncu_full.log 2>&1; echo full=$?
python tools/ncu_summary.py gpurun_out/final2/cfg3_full.ncu-rep gpurun_out/final2/ncu_cfg3_full_summary.json "ncu --set full --clock-control none --import-source on, 1 launch of cf_driver_kernel, cfg3 bf16 (tools/ncu_one.py --config cfg3 --runs 2, launch 2; tools/gpurun/gpu_final2_ncu.sh), round-2 final tree" 2>&1 | tail -2
ls -la gpurun_out/final2/cfg3_full.ncu-rep
