#!/bin/bash
# small-layout (ResNet-20) A/B of env knobs + ncu launch list of the clean bench region
mkdir -p gpurun_out
for cfg in ${CFGS:-"default:" "cap1:CDSGD_SMALL_CTAS_PER_SM=1" "cap1s:CDSGD_SMALL_CTAS_PER_SM=1 CDSGD_STATIC_SCHED=1"}; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 300 python bench.py --workload resnet20 --steps 400 --warmup 20 --no-cpu-baseline --no-e2e --no-secondary --no-self-check > gpurun_out/${TAG}_$name.log 2>&1
  python - gpurun_out/${TAG}_$name.log $name <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-600:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[2], "value", round(d["value"],1), "us/step", round(d["ms_per_step"]*1e3,2), " ".join(f"{k}:{v['avg_us']:.1f}" for k,v in d["kernels"].items()))
PY
done
timeout 300 python bench.py --workload resnet20 --steps 8 --warmup 4 --no-cpu-baseline --no-e2e --no-secondary --no-self-check > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none -k regex:cdsgd -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --workload resnet20 --steps 8 --warmup 4 --no-cpu-baseline --no-e2e --no-secondary --no-self-check > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
