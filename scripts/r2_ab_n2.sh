#!/bin/bash
# N=2 A/B of engine knobs + parity (round 2 development)
mkdir -p gpurun_out
P=29540
timeout 600 python -m pytest tests/test_mgpu.py -q -m gpu -x > gpurun_out/${TAG}_pytest_mgpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_mgpu.log
for cfg in "default:" "pdl_after_ar:CDSGD_PDL_AFTER_AR=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  P=$((P+1))
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 40 --warmup 10 > gpurun_out/${TAG}_bench_${name}.log 2>&1
  echo "$name rc=$?"; grep -o '"value": [0-9.]*' gpurun_out/${TAG}_bench_${name}.log | head -1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((P+5)) scripts/timeline.py --out ${TAG}_timeline_n2 > gpurun_out/${TAG}_timeline.log 2>&1; echo "timeline rc=$?"
