#!/bin/bash
# ncu --set full of the small-layout (ResNet-20) kernels, graph replays, caches not flushed
# (the round's inputs are L2-resident in steady state), then the N=1 sweep
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k "regex:k_fused|k_apply_quant" -s 200 -c 6 \
  -o gpurun_out/${TAG}_r20 python scripts/small_probe.py --periods 10 --reps 20 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}_r20.ncu-rep --page raw --csv > gpurun_out/${TAG}_r20_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_r20.ncu-rep --page details > gpurun_out/${TAG}_r20_details.txt 2>/dev/null
rm -f gpurun_out/${TAG}_r20.ncu-rep
SKIP_MGPU=1 bash scripts/sweep_configs.sh
