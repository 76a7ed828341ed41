python -m pytest tests/test_gpu_engine.py -q -x -k numeric 2>&1 | tail -2
for W in single:262144 single:1048576 single:4194304 resnet20; do
  timeout 300 python bench.py --workload $W --k 4 --steps 24 --warmup 8 --no-cpu-baseline --no-e2e --no-secondary --no-self-check --no-python-ref 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$W', round(d['value'],1), {k:(round(v['avg_us'],1)) for k,v in d['kernels'].items()})"
done
python scripts/small_probe.py --periods 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_step'], d['best_gelem_s'])"
