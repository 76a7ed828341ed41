#!/bin/bash
# ncu --set full of the hot kernels on a short bench (1 GPU). usage: ncu_kernel.sh <tag> [env...]
mkdir -p gpurun_out
TAG=$1; shift
CMD="python bench.py --steps 8 --warmup 4 --no-cpu-baseline --no-e2e --no-secondary"
env "$@" $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
env "$@" ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_quantize|k_apply_quant|k_apply_full|k_fused}" -s ${KSKIP:-6} -c ${KCOUNT:-3} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu $TAG rc=$?"
