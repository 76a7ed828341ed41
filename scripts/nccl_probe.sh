#!/bin/bash
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for N in 2 4 8; do
  [ $N -gt $NG ] && break
  for A in default NVLS Ring; do
    if [ $A = default ]; then unset NCCL_ALGO; else export NCCL_ALGO=$A; fi
    NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 scripts/nccl_probe.py > gpurun_out/nccl_$N_$A.log 2>&1
    echo "N=$N algo=$A rc=$? $(grep '^{' gpurun_out/nccl_$N_$A.log)"
    grep -E "NVLS|nvls" gpurun_out/nccl_$N_$A.log | head -3
  done
done
