#!/bin/bash
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
P=29720
for rep in 1 2; do
for cfg in ${CFGS:-"base:" "arfirst:CDSGD_AR_FIRST=1" "arfirstnopdl:CDSGD_AR_FIRST=1,CDSGD_PLAIN_AFTER_AR=1"}; do
  name=${cfg%%:*}; envs=$(echo ${cfg#*:} | tr ',' ' '); P=$((P+1))
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $P bench.py --gpus $NG --steps 40 --warmup 10 --no-e2e > gpurun_out/${TAG}_bench_${name}.log 2>&1
  python - gpurun_out/${TAG}_bench_${name}.log $name <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); e=d["exchange"]
print(sys.argv[2], "value", round(d["value"],1), " ".join(f"{k}:{v['avg_us']:.1f}/{v['frac']:.2f}" for k,v in d["kernels"].items()), "nccl_ms", round(e.get("nccl_total_ms",0),2), "ok", d["self_check"]["ok"])
PY
done
done
CDSGD_AR_FIRST=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29739 scripts/timeline.py --out ${TAG}_tl > gpurun_out/${TAG}_tl.log 2>&1; echo "timeline rc=$?"
