#!/bin/bash
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l); echo "GPUs: $NG"
timeout 900 python -m pytest tests/test_mgpu.py -x -q -m gpu > gpurun_out/pytest_n8.log 2>&1; echo "mgpu pytest rc=$?"; tail -3 gpurun_out/pytest_n8.log
for N in 4 2; do
for EX in p2p nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N --steps 40 --warmup 10 --exchange $EX > gpurun_out/n8_${N}_$EX.log 2>&1
  python - $N $EX <<'PY'
import json,sys
f=f"gpurun_out/n8_{sys.argv[1]}_{sys.argv[2]}.log"
l=[x for x in open(f) if x.startswith("{")]
if not l: print(sys.argv[1:], open(f).read()[-2500:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.1f}us" for k,v in d["kernels"].items())
x=d['exchange']
print(f"N={sys.argv[1]} {sys.argv[2]:5s} value={d['value']:.1f} step={d['ms_per_step']*1e3:.1f}us e2e={d['e2e']['value']:.1f} {ks} x_us={x and round(x['total_ms']*1e3/x['calls'])} clocks={d['clocks']}")
PY
done
done
