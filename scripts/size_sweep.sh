#!/bin/bash
# N=1 throughput across workloads (ResNet-20/50, VGG-16, single-key 2^16..2^30)
mkdir -p gpurun_out
for W in resnet20 resnet50 vgg16 single:65536 single:1048576 single:16777216 single:268435456 single:1073741824; do
  timeout 300 python bench.py --workload $W --steps 40 --warmup 10 --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/sw.log 2>&1
  python - "$W" <<'PY'
import json,sys
l=[x for x in open("gpurun_out/sw.log") if x.startswith("{")]
if not l: print(sys.argv[1], open("gpurun_out/sw.log").read()[-1200:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.1f}us/{v['frac']:.2f}" for k,v in d["kernels"].items())
print(f"{sys.argv[1]:20s} value={d['value']:8.1f} Gelem/s step={d['ms_per_step']*1e3:9.1f}us  {ks}")
PY
done
