#!/bin/bash
# native symmetric buffers (CUDA IPC): the multi-GPU parity suite + one bench line per N
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_mgpu.py -x -q > gpurun_out/${TAG}_pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -3 gpurun_out/${TAG}_pytest_mgpu.log
NG=$(nvidia-smi -L | wc -l)
for N in 2 4; do
  [ $N -gt $NG ] && break
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2985$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
  python - <<PY
import json
l=[x for x in open("gpurun_out/${TAG}_bench_n$N.log") if x.startswith("{")]
d=json.loads(l[-1]) if l else None
print("N=$N", d and round(d["value"],1), d and d.get("self_check",{}).get("ok")) if d else print(open("gpurun_out/${TAG}_bench_n$N.log").read()[-2000:])
PY
done
