#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in cfg2 cfg3 cfg4; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_$c.log 2>&1
done
