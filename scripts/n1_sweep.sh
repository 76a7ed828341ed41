#!/bin/bash
# N=1 variants of the default bench (plus the GPU test suite first).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_n1s.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_n1s.log
i=0
for v in "$@"; do
  i=$((i+1))
  env $v timeout 300 python bench.py --steps 40 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/n1s_$i.log 2>&1
  python - $i "$v" <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/n1s_{sys.argv[1]}.log") if x.startswith("{")]
if not l: print(sys.argv[2], open(f"gpurun_out/n1s_{sys.argv[1]}.log").read()[-1500:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.1f}us/{v['frac']:.3f}" for k,v in d["kernels"].items())
print(f"{sys.argv[2]:28s} value={d['value']:.1f} step={d['ms_per_step']*1e3:.1f}us  {ks}")
PY
done
