#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
MGRX_VERBOSE=1 timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg4.log
timeout 600 python bench.py --config cfg4 --steps 1 --warmup 0 --impl reference --ref-iters 3 > gpurun_out/bench_cfg4_ref.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
