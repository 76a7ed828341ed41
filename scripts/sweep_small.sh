#!/bin/bash
# re-measure the small-size N=2/4 points of the config sweep (after the copy-engine threshold)
mkdir -p gpurun_out; : > gpurun_out/sweep_small.jsonl
for N in 2 4; do for W in single:1048576 single:16777216; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus $N --workload $W --k 4 --steps 24 --warmup 8 --no-e2e > gpurun_out/sw.log 2>&1
  l=$(grep "^{" gpurun_out/sw.log | tail -1); echo "$l" >> gpurun_out/sweep_small.jsonl
  echo "N=$N $W $(echo "$l" | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")"
done; done
