#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for r in 1 2; do
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/exp_new_r$r.log 2>&1
done
timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/exp_new_cfg4.log 2>&1
echo done
