#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_guard.py tests/test_gpu_fast.py -q -m gpu > gpurun_out/${TAG}_guard.log 2>&1; echo "guard rc=$?"; tail -3 gpurun_out/${TAG}_guard.log
NG=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29581 scripts/nvlink_probe.py --rounds 200 > gpurun_out/${TAG}_nvlink_n$NG.log 2>&1; echo "nvlink rc=$?"; tail -c 1500 gpurun_out/${TAG}_nvlink_n$NG.log
