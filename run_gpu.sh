#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu -x -k "parity or bit_exact or cfg1" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in cfg2; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_$c.log 2>&1
MGRX_AMG_TAIL=2000 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_t2k_$c.log 2>&1
MGRX_AMG_TAIL=0 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_notail_$c.log 2>&1
done
tail -n 3 gpurun_out/pytest_gpu.log
