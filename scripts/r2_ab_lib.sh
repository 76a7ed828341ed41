#!/bin/bash
# A/B of library builds (abvar/*.so) on the N=1 bench: CDSGD_LIB selects the build
mkdir -p gpurun_out
for lib in default ${LIBS}; do
  if [ $lib = default ]; then unset CDSGD_LIB; else export CDSGD_LIB=$PWD/abvar/$lib.so; fi
  for rep in 1 2; do
  timeout 300 python bench.py ${BARGS} --no-cpu-baseline --no-e2e --no-secondary --no-self-check > gpurun_out/${TAG}_$lib.log 2>&1
  python - gpurun_out/${TAG}_$lib.log $lib <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-800:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[2], "value", round(d["value"],1), " ".join(f"{k}:{v['avg_us']:.1f}us/{v['frac']:.3f}" for k,v in d["kernels"].items()))
PY
  done
done
