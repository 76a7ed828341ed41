#!/bin/bash
# BASELINE configs[3] (VGG-16 at 2/4 GPUs, k in {2,4,8}) and configs[4] (gradient-size sweep)
# on one box: one bench JSON line per point into gpurun_out/sweep.jsonl (+ a compact print).
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
NG=$(nvidia-smi -L | wc -l)
run() {  # N workload k
  if [ "$1" -eq 1 ]; then
    timeout 600 python bench.py --workload $2 --k $3 --steps 24 --warmup 8 --no-cpu-baseline --no-e2e --no-secondary --no-self-check > gpurun_out/sw.log 2>&1
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus $1 --workload $2 --k $3 --steps 24 --warmup 8 --no-e2e --no-self-check > gpurun_out/sw.log 2>&1
  fi
  python - "$1" "$2" "$3" <<'PY'
import json,sys
l=[x for x in open("gpurun_out/sw.log") if x.startswith("{")]
if not l: print(sys.argv[1:], open("gpurun_out/sw.log").read()[-600:]); sys.exit()
d=json.loads(l[-1]); open("gpurun_out/sweep.jsonl","a").write(l[-1])
ks=" ".join(f"{k}={v['avg_us']:.0f}us/{v['frac']:.2f}" for k,v in d["kernels"].items())
print(f"N={sys.argv[1]} {sys.argv[2]:18s} k={sys.argv[3]} value={d['value']:8.1f} Gelem/s step={d['ms_per_step']*1e3:9.1f}us {ks}")
PY
}
[ -z "$SKIP_N1" ] && for W in single:65536 single:262144 single:1048576 single:4194304 single:16777216 single:67108864 single:268435456 single:1073741824 resnet20 resnet50 vgg16; do run 1 $W 4; done
[ -z "$SKIP_MGPU" ] && for N in 2 4; do
  [ $N -gt $NG ] && break
  for K in 2 4 8; do run $N vgg16 $K; done
  for W in single:1048576 single:16777216 single:268435456 resnet50; do run $N $W 4; done
done
