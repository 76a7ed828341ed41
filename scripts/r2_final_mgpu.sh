#!/bin/bash
# driver-like: torchrun bench at N=2 and N=4 on a 4-GPU box, reference arm at N=4
mkdir -p gpurun_out
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2975$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29760 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref_n4.log 2>&1; echo "ref N=4 rc=$?"
python - <<PY
import json
for f in ("gpurun_out/${TAG}_bench_n2.log","gpurun_out/${TAG}_bench_n4.log","gpurun_out/${TAG}_ref_n4.log"):
    l=[x for x in open(f) if x.startswith("{")]
    if not l: print(f, open(f).read()[-1500:]); continue
    d=json.loads(l[-1]); print(f, d.get("impl","ours"), "value", round(d["value"],2), "e2e", round(d["e2e"]["value"],2) if d.get("e2e") else None, "selfcheck", (d.get("self_check") or {}).get("ok"))
PY
