#!/bin/bash
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
CDSGD_FUSE_AFTER_AR=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29661 tests/mgpu_check.py p2p > gpurun_out/${TAG}_mgpu.log 2>&1; echo "mgpu fuse rc=$?"; tail -2 gpurun_out/${TAG}_mgpu.log
CFGS="base: fuse:CDSGD_FUSE_AFTER_AR=1 fusence:CDSGD_FUSE_AFTER_AR=1,CDSGD_CE_FRAC=0"
P=29670
for rep in 1 2; do
for cfg in $CFGS; do
  name=${cfg%%:*}; envs=$(echo ${cfg#*:} | tr ',' ' '); P=$((P+1))
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $P bench.py --gpus $NG --steps 40 --warmup 10 --no-e2e --no-self-check > gpurun_out/${TAG}_bench_${name}.log 2>&1
  python - gpurun_out/${TAG}_bench_${name}.log $name <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); e=d["exchange"]
print(sys.argv[2], "value", round(d["value"],1), " ".join(f"{k}:{v['avg_us']:.1f}/{v['frac']:.2f}" for k,v in d["kernels"].items()), "nccl_ms", round(e.get("nccl_total_ms",0),2))
PY
done
done
