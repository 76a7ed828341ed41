#!/bin/bash
# iteration check on one GPU: the GPU suite, the small-layout probe, one bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
O=gpurun_out/${TAG}_small.jsonl; : > $O
timeout 300 python scripts/small_probe.py --periods 1,10 --tag default >> $O 2>>gpurun_out/${TAG}_small.err
timeout 300 python scripts/small_probe.py --periods 10 --weights f32 --tag f32w >> $O 2>>gpurun_out/${TAG}_small.err
timeout 300 python scripts/small_probe.py --layout single:262144 --periods 10 --tag s2p18 >> $O 2>>gpurun_out/${TAG}_small.err
python - <<PY
import json
for l in open("$O"):
    d=json.loads(l); print(d["tag"], {k:round(v,2) for k,v in d["us_per_step"].items()}, round(d["best_gelem_s"],1))
PY
timeout 600 python bench.py --steps 20 --warmup 5 --no-python-ref > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
python - <<PY
import json
l=[x for x in open("gpurun_out/${TAG}_bench.log") if x.startswith("{")]
d=json.loads(l[-1]); print("value",round(d["value"],1),"e2e",round(d["e2e"]["value"],2),{k:(round(v["avg_us"],1),round(v["frac"],3)) for k,v in d["kernels"].items()}, "r20", round(d["secondary"]["resnet20"]["value"],1), round(d["secondary"]["resnet20"]["cuda_graph"]["value"],1), "selfcheck", d.get("self_check",{}).get("ok"))
PY
