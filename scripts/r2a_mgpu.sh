mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2a_gpus.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/r2a_gpus.txt
timeout 900 python -m pytest tests/test_mgpu.py -v -m gpu > gpurun_out/r2a_pytest_mgpu_n2.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2a_pytest_mgpu_n2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 scripts/timeline.py --out r2a_timeline_n2 > gpurun_out/r2a_timeline.log 2>&1; echo "timeline rc=$?"
tail -3 gpurun_out/r2a_timeline.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 40 --warmup 10 > gpurun_out/r2a_bench_n2.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2a_bench_n2.log
