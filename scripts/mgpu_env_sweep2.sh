#!/bin/bash
# N-GPU bench under env variants: bash mgpu_env_sweep.sh N "ENV=..[|bench args]" ...
mkdir -p gpurun_out
N=$1; shift
i=0
for v in "$@"; do
  i=$((i+1))
  envp="${v%%|*}"; argp=""; [[ "$v" == *"|"* ]] && argp="${v#*|}"
  env $envp timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29549 bench.py --gpus $N --steps 40 --warmup 10 --no-e2e $EXTRA $argp > gpurun_out/mes_$i.log 2>&1
  python - $i "$v" <<'PY'
import json,sys
f=f"gpurun_out/mes_{sys.argv[1]}.log"
l=[x for x in open(f) if x.startswith("{")]
if not l: print(sys.argv[2], open(f).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); ks=" ".join(f"{k}={v['avg_us']:.0f}" for k,v in d["kernels"].items())
x=d['exchange'] if d.get('exchange') and 'nccl_calls' in d['exchange'] else None
print(f"{sys.argv[2]:45s} value={d['value']:.1f} step={d['ms_per_step']*1e3:.1f}us {ks} x={x and round(x["nccl_total_ms"]*1e3/x["nccl_calls"])} ar_bus={x and x.get("allreduce_standalone",{}).get("bus_gbs")}")
PY
done
