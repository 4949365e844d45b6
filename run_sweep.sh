#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
PROBE_CFG=cfg4 timeout 600 python tools/probe_spmv.py mgr.0.frelax.amg.1.pre > gpurun_out/probe_ws.log 2>&1 && \
PROBE_CFG=cfg4 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spmv_wspec -c 1 -o gpurun_out/cfg4_wspec_full python tools/probe_spmv.py mgr.0.frelax.amg.1.pre > gpurun_out/ncu_ws.log 2>&1
c=cfg2
rm -f gpurun_out/plan_$c.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_$c.txt python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/prof_plain_$c.log 2>&1 && \
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_$c.txt MGRX_PROFILE_TIMED=1 timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/ncu_$c.log 2>&1
ls -la gpurun_out | tail -8
