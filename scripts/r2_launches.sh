#!/bin/bash
# ncu launch list of the bench command (per-launch duration, serialised, cold-ish caches): the
# kernels' SHARE of a step, to compare with the bench's event-timed roofline kernel
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 8 --warmup 4 --no-secondary --no-python-ref \
  --no-cpu-baseline --no-e2e --no-self-check > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu rc=$?"
python - <<PY
import csv, collections, json
rows=[r for r in csv.DictReader([l for l in open("gpurun_out/${TAG}_launches.csv") if l.startswith('"')])]
tot=collections.Counter(); cnt=collections.Counter()
for r in rows:
    if r.get("Metric Name")!="gpu__time_duration.sum": continue
    k=r["Kernel Name"].split("(")[0][:60]; v=float(r["Metric Value"].replace(",",""))
    unit=r.get("Metric Unit","")
    if unit in ("nsecond","ns"): v/=1000.0
    elif unit in ("msecond","ms"): v*=1000.0
    tot[k]+=v; cnt[k]+=1
s=sum(tot.values())
out={k:{"launches":cnt[k],"total_us":round(tot[k],1),"avg_us":round(tot[k]/cnt[k],2),"share":round(tot[k]/s,4)} for k in tot}
print(json.dumps(out,indent=1))
json.dump(out,open("gpurun_out/${TAG}_launch_shares.json","w"),indent=1)
PY
