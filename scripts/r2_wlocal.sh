#!/bin/bash
# W replica outside the symmetric buffer in p2p mode (default) vs inside (CDSGD_W_SYMMETRIC=1): A/B + parity
mkdir -p gpurun_out
for N in 2 4; do
bash scripts/mgpu_env_sweep2.sh $N "CDSGD_W_SYMMETRIC=1" "CDSGD_W_SYMMETRIC=0" "CDSGD_W_SYMMETRIC=1" "CDSGD_W_SYMMETRIC=0" 2>&1 | tee gpurun_out/r2wl_ab_n$N.txt
for i in 1 2 3 4; do grep -h '^{' gpurun_out/mes_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('N=$N run $i self_check', {k: v for k, v in (d.get('self_check') or {}).items() if k in ('ok','W_bitwise','replicas_bitwise','max_rel_W')})" ; done | tee -a gpurun_out/r2wl_ab_n$N.txt
done
timeout 900 python -m pytest tests/test_mgpu.py -x -q -m gpu > gpurun_out/r2wl_pytest_mgpu.log 2>&1; echo "mgpu pytest rc=$?"; tail -2 gpurun_out/r2wl_pytest_mgpu.log
