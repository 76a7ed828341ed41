#!/bin/bash
# phase probe + small-layout rates (no test suite)
mkdir -p gpurun_out
LIBS=probe TAG=${TAG} bash scripts/r2_probe.sh
O=gpurun_out/${TAG}_small.jsonl; : > $O
timeout 300 python scripts/small_probe.py --periods 1,10 --tag default >> $O 2>>gpurun_out/${TAG}_small.err
timeout 300 python scripts/small_probe.py --layout single:262144 --periods 10 --tag s2p18 >> $O 2>>gpurun_out/${TAG}_small.err
python - <<PY
import json
for l in open("$O"):
    d=json.loads(l); print(d["tag"], {k:round(v,2) for k,v in d["us_per_step"].items()}, round(d["best_gelem_s"],1))
PY
