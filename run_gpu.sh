#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg3.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --sharded --steps 3 --warmup 3 > gpurun_out/bench_sharded1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sharded1.log
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg5.log
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg4.log
tail -n 3 gpurun_out/pytest_gpu.log
