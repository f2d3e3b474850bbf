timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python tools/profile_run.py --fwd-only --out gpurun_out/r2br_prof.json > gpurun_out/r2br_prof.log 2>&1; echo prof rc=$?
timeout 600 python tools/profile_run.py --out gpurun_out/r2br_full.json > gpurun_out/r2br_full.log 2>&1; echo prof rc=$?
