timeout 600 python tools/profile_run.py --out gpurun_out/r2bb_prof.json > gpurun_out/r2bb_prof.log 2>&1; echo rc=$?
