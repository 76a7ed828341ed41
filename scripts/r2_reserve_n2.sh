#!/bin/bash
mkdir -p gpurun_out
P=29560
for cfg in "r0:CDSGD_NCCL_MIN_CTAS=64" "r16:CDSGD_RESERVE_SMS=16 CDSGD_NCCL_MIN_CTAS=16" "r32:CDSGD_RESERVE_SMS=32 CDSGD_NCCL_MIN_CTAS=32" "r24ce0:CDSGD_RESERVE_SMS=24 CDSGD_NCCL_MIN_CTAS=24 CDSGD_CE_FRAC=0" "r48:CDSGD_RESERVE_SMS=48 CDSGD_NCCL_MIN_CTAS=48"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  P=$((P+1))
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1 --master-port $P bench.py --gpus ${NG:-2} --steps 40 --warmup 10 --no-e2e --no-self-check > gpurun_out/${TAG}_bench_${name}.log 2>&1
  echo "$name rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_bench_${name}.log | head -1)"
done
CDSGD_RESERVE_SMS=24 CDSGD_NCCL_MIN_CTAS=24 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1 --master-port $((P+5)) scripts/timeline.py --out ${TAG}_timeline > gpurun_out/${TAG}_timeline.log 2>&1; echo "timeline rc=$?"
