#!/bin/bash
# L2 residency of the small-layout round (ncu without cache flushing, graph replays)
mkdir -p gpurun_out
timeout 600 ncu --cache-control none --clock-control none -k regex:k_ -s 60 -c 8 \
  --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum \
  --csv --log-file gpurun_out/${TAG}_l2.csv python scripts/small_probe.py --periods 10 --reps 20 > gpurun_out/${TAG}_l2.log 2>&1; echo "ncu rc=$?"
python - <<PY
import csv
rows=list(csv.DictReader([l for l in open("gpurun_out/${TAG}_l2.csv") if l.startswith('"')]))
for r in rows:
    print(r["ID"], r["Kernel Name"][:40], r["Metric Name"], r["Metric Value"])
PY
