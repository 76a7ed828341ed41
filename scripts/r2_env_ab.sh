#!/bin/bash
# N=1 A/B of env knobs on a workload: CFGS="name:ENV=.. name2:..." WL=resnet20|resnet50
mkdir -p gpurun_out
WL=${WL:-resnet50}; ST=${ST:-40}
for rep in 1 2; do
for cfg in $CFGS; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 300 python bench.py --workload $WL --steps $ST --warmup 20 --no-cpu-baseline --no-e2e --no-secondary --no-self-check > gpurun_out/${TAG}_$name.log 2>&1
  python - gpurun_out/${TAG}_$name.log $name <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-600:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[2], "value", round(d["value"],1), "us/step", round(d["ms_per_step"]*1e3,2), " ".join(f"{k}:{v['avg_us']:.1f}/{v['frac']:.3f}" for k,v in d["kernels"].items()))
PY
done
done
