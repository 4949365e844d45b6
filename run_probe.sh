#!/bin/bash
mkdir -p gpurun_out
for r in 1 2 3; do
MGRX_VERBOSE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bv_$r.json 2>gpurun_out/bv_$r.err
done
echo done
