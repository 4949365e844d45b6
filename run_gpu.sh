#!/bin/bash
# round-1 re-entry sanity: GPU parity tests, default bench, cfg3/cfg4 re-measure
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg3.log
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg4.log
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log
