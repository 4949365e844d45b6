#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for g in 0 1; do for c in cfg2 cfg4; do
MGRX_SPMV_GEOM=$g timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/exp_g${g}_$c.log 2>&1
done; done
echo done
