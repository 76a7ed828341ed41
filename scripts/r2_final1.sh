#!/bin/bash
# driver-like sequence on 1 GPU: GPU tests, smoke, bench (default), reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_n1.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref_n1.log 2>&1; echo "ref rc=$?"
python - <<PY
import json
for f in ("gpurun_out/${TAG}_bench_n1.log", "gpurun_out/${TAG}_ref_n1.log"):
    l=[x for x in open(f) if x.startswith("{")]
    if not l: print(f, open(f).read()[-2000:]); continue
    d=json.loads(l[-1]); print(f, d.get("impl","ours"), "value", round(d["value"],3), "e2e", d["e2e"]["value"] if d.get("e2e") else None)
    if "self_check" in d: print("  self_check ok", d["self_check"]["ok"], "W_bitwise", d["self_check"].get("W_bitwise"))
    if d.get("python_reference"): print("  python ref", {k: (v.get("value") if isinstance(v, dict) else v) for k, v in d["python_reference"].items()})
PY
