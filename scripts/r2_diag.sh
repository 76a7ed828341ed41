#!/bin/bash
# final suite on a 4-GPU box + where F's extra time at N>1 goes (diagnostic knobs: wrong results, timing only)
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2dg_gpus.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2dg_pytest_gpu.log 2>&1; echo "gpu pytest rc=$?"; tail -2 gpurun_out/r2dg_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2dg_smoke.log 2>&1; tail -1 gpurun_out/r2dg_smoke.log
for N in 2 4; do
bash scripts/mgpu_env_sweep2.sh $N "CDSGD_DIAG_NONE=1|--no-self-check" "CDSGD_DIAG_NO_WAIT=1|--no-self-check" "CDSGD_DIAG_NO_REMOTE_CODES=1|--no-self-check" "CDSGD_DIAG_NO_WAIT=1 CDSGD_DIAG_NO_REMOTE_CODES=1|--no-self-check" 2>&1 | tee gpurun_out/r2dg_diag_n$N.txt
done
