#!/bin/bash
# 1 GPU: GPU test suite, default bench line, then the ncu kernel captures (round 2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu ${PYARGS} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
python - gpurun_out/${TAG}_bench.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(open(sys.argv[1]).read()[-3000:]); sys.exit()
d=json.loads(l[-1]); print(" value", round(d["value"],1), "ms/step", round(d["ms_per_step"]*1e3,1), "e2e", round(d["e2e"]["value"],2))
for k,v in d["kernels"].items(): print("   ", k, round(v["avg_us"],1), "us", round(v["frac"],3))
print("  self_check", d["self_check"]); print("  secondary", json.dumps(d["secondary"])[:1500]); print("  cpu", json.dumps(d["cpu_baseline"])[:1500])
PY
[ -n "$NCU" ] && TAG=${TAG}ncu bash scripts/r2_ncu.sh
