#!/bin/bash
# A/B of the merged Arnoldi phase: GPU parity suite, full-size parity, cfg2
# bench with the merge on and off (MGRX_ARNOLDI_MERGE=0), cfg3-5 benches.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_m1.log 2>&1
MGRX_ARNOLDI_MERGE=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_m0.log 2>&1
for c in cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_$c.log 2>&1; done
MGRX_ARNOLDI_MERGE=0 timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_cfg3_m0.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/pytest_full.log
