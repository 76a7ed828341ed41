#!/bin/bash
# standalone kernel timings + one ncu --set full capture per hot kernel (ResNet-50 layout)
mkdir -p gpurun_out
W=${WEIGHTS:-f64}
timeout 300 python scripts/kernel_probe.py --weights $W --nranks 1,2,4,8 --reps 20 > gpurun_out/${TAG}_probe.jsonl 2>&1; echo "probe rc=$?"
cat gpurun_out/${TAG}_probe.jsonl
for spec in "K1:1:k_quantize_tma" "F:1:k_fused_ldg" "F:4:k_fused_ldg" "K2:1:k_apply_quant" "K2:4:k_apply_quant" "K3:4:k_apply_full_tma"; do
  IFS=: read only nr kern <<< "$spec"
  timeout 300 python scripts/kernel_probe.py --weights $W --only $only --nranks $nr --reps 1 > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -s 3 -c 1 \
      -o gpurun_out/${TAG}_${only}_n${nr} python scripts/kernel_probe.py --weights $W --only $only --nranks $nr --reps 1 \
      > gpurun_out/${TAG}_${only}_n${nr}.ncu.log 2>&1
  echo "ncu $spec rc=$?"
  # keep the report small enough to travel back: raw metrics as CSV, details page as text
  ncu -i gpurun_out/${TAG}_${only}_n${nr}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${only}_n${nr}.raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${only}_n${nr}.ncu-rep --page details > gpurun_out/${TAG}_${only}_n${nr}.details.txt 2>/dev/null
  rm -f gpurun_out/${TAG}_${only}_n${nr}.ncu-rep
done
