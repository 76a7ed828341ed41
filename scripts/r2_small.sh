#!/bin/bash
# small-layout latency probe: knob variants, then one ncu --set full of the ResNet-20 fused kernel
mkdir -p gpurun_out
O=gpurun_out/${TAG}_small.jsonl; : > $O
P="python scripts/small_probe.py --periods 1,10"
timeout 300 $P --floor --tag default >> $O 2>gpurun_out/${TAG}_small.err
CDSGD_NO_PDL=1 timeout 300 $P --tag nopdl >> $O 2>>gpurun_out/${TAG}_small.err
CDSGD_SMALL_CTAS_PER_SM=1 timeout 300 $P --tag cap1 >> $O 2>>gpurun_out/${TAG}_small.err
CDSGD_CH1_TPW=0 timeout 300 $P --tag noch1 >> $O 2>>gpurun_out/${TAG}_small.err
CDSGD_NO_TILE_TABLE=1 timeout 300 $P --tag notab >> $O 2>>gpurun_out/${TAG}_small.err
timeout 300 $P --weights f32 --tag f32w >> $O 2>>gpurun_out/${TAG}_small.err
timeout 300 python scripts/small_probe.py --layout single:262144 --periods 10 --tag s2p18 >> $O 2>>gpurun_out/${TAG}_small.err
python - <<PY
import json
for l in open("$O"):
    d=json.loads(l); print(d["tag"], {k:round(v,2) for k,v in d["us_per_step"].items()}, round(d["best_gelem_s"],1), d.get("us_per_tiny_kernel_in_graph"))
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 40 -c 4 -o gpurun_out/${TAG}_r20 python scripts/small_probe.py --periods 10 --reps 10 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
for f in gpurun_out/${TAG}_r20.ncu-rep; do
  ncu -i $f --page raw --csv > gpurun_out/${TAG}_r20_raw.csv 2>/dev/null
  ncu -i $f --page details > gpurun_out/${TAG}_r20_details.txt 2>/dev/null
  ncu -i $f --page source --csv > gpurun_out/${TAG}_r20_source.csv 2>/dev/null
  rm -f $f
done
ls -la gpurun_out/${TAG}_*
