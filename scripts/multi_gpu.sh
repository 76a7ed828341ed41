#!/bin/bash
# Multi-GPU checks on one box: GPU test suite (incl. torchrun parity), then bench at N=1..NGPU.
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
echo "GPUs: $NG"
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_mgpu.log
for N in 1 2 4 8; do
  [ $N -gt $NG ] && break
  if [ $N -eq 1 ]; then
    timeout 300 python bench.py --steps 40 --warmup 10 --no-cpu-baseline > gpurun_out/bench_n$N.log 2>&1
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus $N --steps 40 --warmup 10 $EXTRA > gpurun_out/bench_n$N.log 2>&1
  fi
  echo "bench N=$N rc=$?"
  python - $N <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/bench_n{sys.argv[1]}.log") if x.startswith("{")]
if not l: print(open(f"gpurun_out/bench_n{sys.argv[1]}.log").read()[-3000:]); sys.exit()
d=json.loads(l[-1]); print("  value", round(d["value"],1), "Gelem/s  ms/step", round(d["ms_per_step"]*1e3,1), "us  e2e", d["e2e"] and round(d["e2e"]["value"],1))
for k,v in d["kernels"].items(): print("    ", k, round(v["avg_us"],1), "us", round(v["achieved_gbs"]), "GB/s", round(v["frac"],3))
print("   exchange", d.get("exchange"))
PY
done
