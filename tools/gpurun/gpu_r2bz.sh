timeout 900 python tools/profile_run.py --config cfg4 --T 1000 --stack-budget 33600000000 --swap-smallest-first --out gpurun_out/r2bz_swap.json > gpurun_out/r2bz_swap.log 2>&1; echo rc=$?
timeout 900 python tools/profile_run.py --config cfg4 --T 1000 --out gpurun_out/r2bz_noswap.json > gpurun_out/r2bz_noswap.log 2>&1; echo rc=$?
