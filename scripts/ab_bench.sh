#!/bin/bash
# A/B of kernel variants on the default bench (ResNet-50, N=1), plus the GPU test suite.
# usage: bash scripts/ab_bench.sh "ENV=.. ENV2=.." "..."   (each arg = one variant's env)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
i=0
for v in "$@"; do
  i=$((i+1))
  env $v timeout 300 python bench.py --steps 40 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$i.log 2>&1
  echo "[$v] rc=$?"
  python - "$i" <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/bench_v{sys.argv[1]}.log") if x.startswith("{")]
if not l: print(open(f"gpurun_out/bench_v{sys.argv[1]}.log").read()[-2000:]); sys.exit()
d=json.loads(l[-1]); print("  value", round(d["value"],1), "ms/step", round(d["ms_per_step"]*1e3,1), "us")
for k,v in d["kernels"].items(): print("    ", k, round(v["avg_us"],1), "us", round(v["achieved_gbs"]), "GB/s", round(v["frac"],3))
PY
done
