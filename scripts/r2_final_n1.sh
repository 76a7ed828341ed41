#!/bin/bash
# driver-like N=1 sequence: GPU suite, smoke, reference arm, bench (default flags)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
python - <<PY
import json
for f in ("gpurun_out/${TAG}_ref.log","gpurun_out/${TAG}_bench.log"):
    l=[x for x in open(f) if x.startswith("{")]
    d=json.loads(l[-1]); print(f, d.get("impl","ours"), "value", round(d["value"],2), "e2e", round(d["e2e"]["value"],2), "clocks", d.get("clocks"))
    if "secondary" in d:
        r=d["secondary"]["resnet20"]; print("  r20 host", round(r["value"],1), "graph", round(r["cuda_graph"]["value"],1), "graph1", round(r["cuda_graph"]["one_period_per_graph"]["value"],1), "cold", round(r["cold_l2"]["value"],1), "cold graph", r["cold_l2"].get("cuda_graph"))
        print("  roofline", d["roofline"], "selfcheck", d.get("self_check",{}).get("ok"))
PY
