#!/bin/bash
# round 2: launch lists of one timed solve per config (SpMV plans replayed
# from a plain run), plus a plain bench line per config
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in ${CONFIGS:-cfg2 cfg3 cfg4 cfg5}; do
rm -f gpurun_out/plan_$c.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_$c.txt timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_$c.log 2>&1
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_$c.txt MGRX_PROFILE_TIMED=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/ncu_$c.log 2>&1
python tools/launch_stats.py gpurun_out/launches_$c.csv > gpurun_out/shares_$c.txt 2>&1
done
tail -n 3 gpurun_out/bench_*.log | cut -c1-600; head -n 12 gpurun_out/shares_*.txt
