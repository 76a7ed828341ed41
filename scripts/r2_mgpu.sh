#!/bin/bash
# N-GPU: multi-GPU parity suite + bench line + timeline (round 2). NG = GPUs on the box.
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${TAG}_gpus.txt
timeout 1200 python -m pytest tests/test_mgpu.py -v -m gpu > gpurun_out/${TAG}_pytest_mgpu.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/${TAG}_pytest_mgpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG ${BARGS} > gpurun_out/${TAG}_bench_n$NG.log 2>&1; echo "bench rc=$?"
python - gpurun_out/${TAG}_bench_n$NG.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(open(sys.argv[1]).read()[-2000:]); sys.exit()
d=json.loads(l[-1]); print(" value", round(d["value"],1), "ms/step", round(d["ms_per_step"]*1e3,1), "e2e", round(d["e2e"]["value"],2))
for k,v in d["kernels"].items(): print("   ", k, round(v["avg_us"],1), "us", round(v["frac"],3))
print("  exchange", json.dumps(d["exchange"]))
print("  self_check", d["self_check"])
PY
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29572 scripts/timeline.py --out ${TAG}_timeline_n$NG > gpurun_out/${TAG}_timeline.log 2>&1; echo "timeline rc=$?"
