#!/bin/bash
# split correction apply (K3 on NCCL's share first): multi-GPU parity suite + A/B at N=4 / N=2
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2sp_gpus.txt
timeout 900 python -m pytest tests/test_mgpu.py -x -q -m gpu > gpurun_out/r2sp_pytest_mgpu.log 2>&1; echo "mgpu pytest rc=$?"; tail -2 gpurun_out/r2sp_pytest_mgpu.log
bash scripts/mgpu_env_sweep2.sh 4 "CDSGD_SPLIT_APPLY=0" "CDSGD_SPLIT_APPLY=1" "CDSGD_SPLIT_APPLY=0" "CDSGD_SPLIT_APPLY=1" 2>&1 | tee gpurun_out/r2sp_ab_n4.txt
bash scripts/mgpu_env_sweep2.sh 2 "CDSGD_SPLIT_APPLY=0" "CDSGD_SPLIT_APPLY=1" 2>&1 | tee gpurun_out/r2sp_ab_n2.txt
