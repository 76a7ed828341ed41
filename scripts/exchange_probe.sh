#!/bin/bash
# Isolate round types at N=$1: k=1000 (compressed only) vs k=1 (correction only), p2p vs nccl.
mkdir -p gpurun_out
N=${1:-4}
for EX in p2p nccl; do
  for K in 1000 4 1; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus $N --steps 40 --warmup 10 --k $K --exchange $EX --no-e2e --no-cpu-baseline > gpurun_out/xp_${EX}_$K.log 2>&1
    python - $EX $K <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/xp_{sys.argv[1]}_{sys.argv[2]}.log") if x.startswith("{")]
if not l: print(sys.argv[1:], open(f"gpurun_out/xp_{sys.argv[1]}_{sys.argv[2]}.log").read()[-1500:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.0f}" for k,v in d["kernels"].items())
x=d.get("exchange") or {}
print(f"{sys.argv[1]:5s} k={sys.argv[2]:5s} value={d['value']:.1f} step={d['ms_per_step']*1e3:.1f}us  {ks}  xcalls={x.get('calls')} x_us={x and x['nccl_total_ms']*1e3/max(1,x['nccl_calls']):.0f}")
PY
  done
done
