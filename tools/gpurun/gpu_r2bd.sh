timeout 600 python tools/profile_run.py --fwd-only --out gpurun_out/r2bn_prof.json > gpurun_out/r2bn_prof.log 2>&1; echo prof rc=$?
timeout 600 python tools/profile_run.py --fwd-only --no-tiles --out gpurun_out/r2bn_nt.json > gpurun_out/r2bn_nt.log 2>&1; echo prof rc=$?
