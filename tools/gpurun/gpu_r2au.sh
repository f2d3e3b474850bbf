python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2au_build.log 2>&1
mkdir -p gpurun_out/sanitizer
timeout 1500 compute-sanitizer --tool memcheck --launch-timeout 0 --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer/memcheck.log 2>&1; echo "memcheck rc=$?"
tail -5 gpurun_out/sanitizer/memcheck.log
timeout 1500 compute-sanitizer --tool synccheck --launch-timeout 0 --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer/synccheck.log 2>&1; echo "synccheck rc=$?"
tail -5 gpurun_out/sanitizer/synccheck.log
