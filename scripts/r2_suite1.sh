#!/bin/bash
# 1-GPU: full GPU test suite + default bench line + reference arm (round 2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu ${PYARGS} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc=$?"
tail -c 300 gpurun_out/${TAG}_ref.log
