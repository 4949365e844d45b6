#!/bin/bash
# launch list of one timed solve (host-driven GMRES loop: ncu does not see inside
# the conditional-graph cycle), SpMV choices replayed from a plain run
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in ${CONFIGS:-cfg2}; do
rm -f gpurun_out/plan_$c.txt
MGRX_GMRES_GRAPH=0 MGRX_SPMV_PLAN_FILE=gpurun_out/plan_$c.txt timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_plain_$c.log 2>&1
MGRX_GMRES_GRAPH=0 MGRX_SPMV_PLAN_FILE=gpurun_out/plan_$c.txt MGRX_PROFILE_TIMED=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/ncu_$c.log 2>&1
python tools/launch_stats.py gpurun_out/launches_$c.csv > gpurun_out/shares_$c.txt 2>&1
grep '^{' gpurun_out/bench_plain_$c.log | tail -n 1 | cut -c1-300
cat gpurun_out/shares_$c.txt
done
