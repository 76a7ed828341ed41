#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fused.log
i=0
for v in "X=1" "CDSGD_FUSED_CFG=12x2" "CDSGD_FUSED_CFG=6x2" "CDSGD_FUSED_CFG=8x3" "CDSGD_NO_FUSE=1"; do
  i=$((i+1))
  env $v timeout 300 python bench.py --steps 40 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/fs_$i.log 2>&1
  python - $i "$v" <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/fs_{sys.argv[1]}.log") if x.startswith("{")]
if not l: print(sys.argv[2], open(f"gpurun_out/fs_{sys.argv[1]}.log").read()[-1500:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.1f}us/{v['frac']:.3f}" for k,v in d["kernels"].items())
print(f"N=1 {sys.argv[2]:24s} value={d['value']:.1f} step={d['ms_per_step']*1e3:.1f}us  {ks}")
PY
done
for EX in p2p nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29539 bench.py --gpus 2 --steps 40 --warmup 10 --exchange $EX --no-e2e > gpurun_out/fs2_$EX.log 2>&1
  python - $EX <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/fs2_{sys.argv[1]}.log") if x.startswith("{")]
if not l: print(sys.argv[1], open(f"gpurun_out/fs2_{sys.argv[1]}.log").read()[-2500:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.1f}us" for k,v in d["kernels"].items())
print(f"N=2 {sys.argv[1]:5s} value={d['value']:.1f} step={d['ms_per_step']*1e3:.1f}us  {ks} x={d['exchange'] and round(d['exchange']['total_ms']*1e3/d['exchange']['calls'])}")
PY
done
