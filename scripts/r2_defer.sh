#!/bin/bash
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_mgpu.py -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
CFGS="defer: nodefer:CDSGD_CE_DEFER=0" TAG=${TAG}b bash scripts/r2_arfirst.sh
