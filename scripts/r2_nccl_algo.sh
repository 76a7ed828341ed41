#!/bin/bash
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29701 scripts/nccl_probe.py > gpurun_out/${TAG}_nccl_n$NG.log 2>&1
echo "rc=$?"; grep -E "^\{" gpurun_out/${TAG}_nccl_n$NG.log; grep -iE "AllReduce.*(Ring|Tree|NVLS|CollNet)|algorithm|NVLS" gpurun_out/${TAG}_nccl_n$NG.log | head -12
