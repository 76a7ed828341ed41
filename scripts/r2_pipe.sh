#!/bin/bash
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python scripts/pipeline_probe.py --out gpurun_out/${TAG}_pipe_n1.json > gpurun_out/${TAG}_pipe_n1.log 2>&1; echo "pipe n1 rc=$?"; tail -c 800 gpurun_out/${TAG}_pipe_n1.log
if [ $NG -gt 1 ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29641 scripts/pipeline_probe.py --out gpurun_out/${TAG}_pipe_n$NG.json > gpurun_out/${TAG}_pipe_n$NG.log 2>&1; echo "pipe n$NG rc=$?"; tail -c 800 gpurun_out/${TAG}_pipe_n$NG.log
fi
