#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
MGRX_PDL=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bp_trig_$r.json 2>&1
MGRX_LIB=$PWD/variants/libmgrx_notrig.so MGRX_PDL=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bp_notrig_$r.json 2>&1
MGRX_PDL=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bp_off_$r.json 2>&1
done
echo done
