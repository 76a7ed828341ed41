#!/bin/bash
# copy-engine phase flags by stream memory operations: parity suite, then A/B at N=4 and N=2
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_mgpu.py -x -q > gpurun_out/${TAG}_pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -2 gpurun_out/${TAG}_pytest_mgpu.log
bash scripts/mgpu_env_sweep2.sh 4 "X=1" "CDSGD_FLAG_MEMOPS=0" "X=2" "CDSGD_FLAG_MEMOPS=0 X=2" 2>&1 | grep "value="
bash scripts/mgpu_env_sweep2.sh 2 "X=1" "CDSGD_FLAG_MEMOPS=0" 2>&1 | grep "value="
