# 2 GPUs: DP bench debug (short watchdog, small T first)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1
BENCH_DEBUG=1 timeout 200 python bench.py --gpus 2 --parallel dp --T 8 --steps 2 --warmup 3 --no-cpu-baseline --watchdog-ms 20000 > gpurun_out/r2h_dp_T8.log 2>&1
echo "dp T8 exit $?"
BENCH_DEBUG=1 timeout 200 python bench.py --gpus 2 --parallel dp --config cfg2 --steps 2 --warmup 3 --no-cpu-baseline --watchdog-ms 20000 > gpurun_out/r2h_dp_cfg2.log 2>&1
echo "dp cfg2 exit $?"
BENCH_DEBUG=1 timeout 300 python bench.py --gpus 2 --parallel dp --steps 5 --warmup 3 --no-cpu-baseline --watchdog-ms 30000 > gpurun_out/r2h_dp_cfg3.log 2>&1
echo "dp cfg3 exit $?"
grep -h "metric\|Error\|error\|ms=" gpurun_out/r2h_dp_*.log | cut -c1-300
