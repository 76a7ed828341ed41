#!/bin/bash
mkdir -p gpurun_out
N=${1:-4}
for A in "default" "allreduce:nvls" "allreduce:nvlstree" "allreduce:tree"; do
  if [ "$A" = default ]; then unset NCCL_ALGO; else export NCCL_ALGO="$A"; fi
  NCCL_DEBUG=WARN timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29537 scripts/nccl_probe.py > gpurun_out/nvls_probe.log 2>&1
  echo "N=$N ALGO=$A rc=$? $(grep '^{' gpurun_out/nvls_probe.log)"
  grep -E "NCCL WARN" gpurun_out/nvls_probe.log | head -2
done
