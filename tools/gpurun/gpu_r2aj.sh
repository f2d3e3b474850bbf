timeout 600 python tools/profile_run.py --out gpurun_out/r2aj_prof.json > gpurun_out/r2aj_prof.log 2>&1
head -60 gpurun_out/r2aj_prof.log | grep -v "^ *\"[A-Z_]*\": {$" | head -60
