#!/bin/bash
# launch lists of one timed solve (cfg2 / cfg3 / cfg4 default strategies), SpMV
# staged/direct choices replayed from a plain run (ncu distorts the setup timing)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in cfg2 cfg3 cfg4; do
rm -f gpurun_out/plan_$c.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_$c.txt python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/prof_plain_$c.log 2>&1 && \
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_$c.txt MGRX_PROFILE_TIMED=1 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/ncu_$c.log 2>&1
done
MGRX_GMRES_PROF=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_steps.log 2>&1
echo done
