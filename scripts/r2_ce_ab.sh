#!/bin/bash
# copy-engine share of the correction all-reduce: parallel per-peer copies vs serial, split fractions
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_mgpu.py -q -m gpu -k "copy_engine or engine_parity" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
P=29620
for cfg in ${CFGS:-"par:" "serial:CDSGD_CE_SERIAL=1" "par70:CDSGD_CE_FRAC=0.7" "par85:CDSGD_CE_FRAC=0.85" "par100:CDSGD_CE_FRAC=1.0"}; do
  name=${cfg%%:*}; envs=${cfg#*:}; P=$((P+1))
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $P bench.py --gpus $NG --steps 40 --warmup 10 --no-e2e --no-self-check > gpurun_out/${TAG}_bench_${name}.log 2>&1
  python - gpurun_out/${TAG}_bench_${name}.log $name <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); e=d["exchange"]
print(sys.argv[2], "value", round(d["value"],1), " ".join(f"{k}:{v['avg_us']:.1f}/{v['frac']:.2f}" for k,v in d["kernels"].items()),
      "nccl_ms", round(e.get("nccl_total_ms",0),2), "ce_ms", round(e.get("ce_total_ms",0),2))
PY
done
