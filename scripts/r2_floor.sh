#!/bin/bash
mkdir -p gpurun_out
for c in 284 148 74; do ./scripts/launch_floor $c; done > gpurun_out/${TAG}_floor.jsonl 2>&1; cat gpurun_out/${TAG}_floor.jsonl
O=gpurun_out/${TAG}_small.jsonl; : > $O
timeout 300 python scripts/small_probe.py --periods 10 --tag default >> $O 2>>gpurun_out/${TAG}_small.err
python - <<PY
import json
for l in open("$O"):
    d=json.loads(l); print(d["tag"], {k:round(v,2) for k,v in d["us_per_step"].items()}, round(d["best_gelem_s"],1))
PY
timeout 600 python bench.py --steps 20 --warmup 5 --no-python-ref --no-self-check --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
python - <<PY
import json
l=[x for x in open("gpurun_out/${TAG}_bench.log") if x.startswith("{")]
d=json.loads(l[-1]); print("value",round(d["value"],1),{k:(round(v["avg_us"],1),round(v["frac"],3)) for k,v in d["kernels"].items()}, "r20", round(d["secondary"]["resnet20"]["value"],1), round(d["secondary"]["resnet20"]["cuda_graph"]["value"],1))
PY
