#!/bin/bash
mkdir -p gpurun_out
N=${1:-2}
for K in 1 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus $N --steps 40 --warmup 10 --k $K --no-e2e > gpurun_out/pp_$K.log 2>&1
  python - $K <<'PY'
import json,sys
f=f"gpurun_out/pp_{sys.argv[1]}.log"
l=[x for x in open(f) if x.startswith("{")]
if not l: print(open(f).read()[-2500:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.1f}us" for k,v in d["kernels"].items())
print(f"k={sys.argv[1]} value={d['value']:.1f} step={d['ms_per_step']*1e3:.1f}us {ks} waits={d.get('waits')}")
PY
done
