#!/bin/bash
# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md), on the single-GPU suite minus the
# full-size (25.6M-element) cases, which the instrumentation would slow to hours.
mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
SEL=${SEL:-"tests/test_gpu_codec.py tests/test_gpu_engine.py tests/test_gpu_config_i.py tests/test_gpu_fast.py"}
KEXPR=${KEXPR:-"not resnet50 and not full and not 1M and not 1048575 and not drift and not 3_000_000"}
timeout ${TLIM:-1500} compute-sanitizer --tool $TOOL ${SANARGS} --error-exitcode 17 --print-limit 50 \
    python -m pytest $SEL -q -x -k "$KEXPR" -p no:cacheprovider > gpurun_out/${TAG}_${TOOL}.log 2>&1
echo "sanitizer $TOOL rc=$?"
grep -E "ERROR SUMMARY|passed|failed|Error" gpurun_out/${TAG}_${TOOL}.log | tail -8
