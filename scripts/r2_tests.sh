#!/bin/bash
# GPU test suite on this box (N GPUs), logs under gpurun_out/ with prefix $TAG
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpus.txt
timeout 1500 python -m pytest tests -q -m gpu -x ${PYARGS} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/${TAG}_pytest.log
