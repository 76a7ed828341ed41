#!/bin/bash
mkdir -p gpurun_out
C="python bench.py --workload resnet20 --steps 8 --warmup 4 --no-cpu-baseline --no-e2e --no-secondary --no-self-check"
timeout 300 $C > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__cycles_active.avg,sm__cycles_elapsed.avg --clock-control none -k regex:k_ -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv $C > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
