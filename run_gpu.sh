#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
MGRX_VERBOSE=1 timeout 900 python bench.py --config cfg3 --steps 2 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg3.log
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 3 --impl reference --ref-iters 5 > gpurun_out/bench_cfg3_ref.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
