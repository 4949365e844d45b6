#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for r in 1 2; do
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/exp_row4_r$r.log 2>&1
MGRX_LIB=$PWD/libmgrx_row8.so timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/exp_row8_r$r.log 2>&1
done
MGRX_LIB=$PWD/libmgrx_row8.so timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/exp_row8_cfg3.log 2>&1
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/exp_row4_cfg3.log 2>&1
echo done
