#!/bin/bash
# 4-GPU verification: the multi-GPU parity suite, then the driver-like bench lines
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/${TAG}_gpus.txt
timeout 1800 python -m pytest tests/test_mgpu.py -x -q > gpurun_out/${TAG}_pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -3 gpurun_out/${TAG}_pytest_mgpu.log
TAG=${TAG} bash scripts/r2_final_mgpu.sh
