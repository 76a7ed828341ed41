#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x ${PYARGS} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/${TAG}_pytest.log
for w in f64 f32; do
timeout 600 python bench.py --weights $w --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.log 2>&1; echo "bench $w rc=$?"
python - $w <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/{sys.argv[0] if False else ''}{__import__('os').environ.get('TAG')}_bench_{sys.argv[1]}.log") if x.startswith("{")]
d=json.loads(l[-1]); print(" value", round(d["value"],1), "ms/step", round(d["ms_per_step"]*1e3,1), "us", "e2e", round(d["e2e"]["value"],2))
for k,v in d["kernels"].items(): print("   ", k, round(v["avg_us"],1), "us", round(v["frac"],3))
print("  self_check", d["self_check"])
print("  r20", d["secondary"]["resnet20"]["value"], d["secondary"]["resnet20"]["cold_l2"]["value"])
PY
done
