timeout 900 python tools/profile_run.py --config cfg5 --out gpurun_out/r2bi_prof.json > gpurun_out/r2bi_prof.log 2>&1; echo rc=$?
