#!/bin/bash
# multi-GPU: parity suite (torchrun, all exchanges) + bench per exchange mode at N=NGPU and 2
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l); echo "GPUs: $NG"
timeout 1200 python -m pytest tests/test_mgpu.py -x -q -m gpu > gpurun_out/pytest_n8.log 2>&1; echo "mgpu pytest rc=$?"; tail -3 gpurun_out/pytest_n8.log
for N in $NG 2; do
for EX in p2p p2p-exact nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N --steps 40 --warmup 10 --exchange $EX --no-e2e > gpurun_out/n8_${N}_$EX.log 2>&1
  python - $N $EX <<'PY'
import json,sys
f=f"gpurun_out/n8_{sys.argv[1]}_{sys.argv[2]}.log"
l=[x for x in open(f) if x.startswith("{")]
if not l: print(sys.argv[1:], open(f).read()[-2500:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.1f}us" for k,v in d["kernels"].items())
x=d['exchange'] if d.get('exchange') and 'nccl_calls' in d['exchange'] else None
print(f"N={sys.argv[1]} {sys.argv[2]:9s} value={d['value']:.1f} step={d['ms_per_step']*1e3:.1f}us {ks} x_us={x and round(x['nccl_total_ms']*1e3/x['nccl_calls'])} waits={d.get('waits')}")
PY
done
done
