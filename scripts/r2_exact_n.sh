#!/bin/bash
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
P=29690
for ex in p2p-exact p2p; do
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $P bench.py --gpus $NG --exchange $ex --no-e2e > gpurun_out/${TAG}_bench_$ex.log 2>&1
  python - gpurun_out/${TAG}_bench_$ex.log $ex <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1])
print(sys.argv[2], "value", round(d["value"],1), " ".join(f"{k}:{v['avg_us']:.1f}/{v['frac']:.2f}" for k,v in d["kernels"].items()), "selfcheck", {k: d["self_check"].get(k) for k in ("ok","W_bitwise","W_max_abs_err","replicas_bitwise_equal")})
PY
done
