#!/bin/bash
# bench (plain) -> ncu launch list of the same command -> ncu --set full of the persistent kernel
set -x
mkdir -p gpurun_out
CMD="python bench.py --config cfg3 --precision bf16 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$?
CMD2="python tools/ncu_one.py --config cfg3 --runs 2"
$CMD2 > gpurun_out/ncu_one_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cf_driver -s 1 -c 1 -o gpurun_out/cfg3_full $CMD2 > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
