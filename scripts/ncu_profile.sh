#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): launch list + ncu --set full of K1/K2/K3.
mkdir -p gpurun_out
set -x
CMD="python bench.py --steps 8 --warmup 4 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/plain_small2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_quantize|k_apply_quant|k_apply_full" -s 6 -c 3 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
