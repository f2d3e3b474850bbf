for w in 147 96 48 24; do
timeout 600 python tools/profile_run.py --fwd-only --workers $w --out gpurun_out/r2bk_w$w.json > gpurun_out/r2bk_w$w.log 2>&1; echo w=$w rc=$?
done
