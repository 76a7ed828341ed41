#!/bin/bash
mkdir -p gpurun_out
N=${1:-2}
for A in "allreduce:nvls" "allreduce:nvls;allgather:ring" "NVLS"; do
  NCCL_ALGO="$A" NCCL_DEBUG=WARN timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29537 scripts/nccl_probe.py > gpurun_out/nvls_probe.log 2>&1
  echo "ALGO=$A rc=$? $(grep '^{' gpurun_out/nvls_probe.log)"
  grep -iE "warn|error|invalid" gpurun_out/nvls_probe.log | grep -v "^W1018" | head -6
done
