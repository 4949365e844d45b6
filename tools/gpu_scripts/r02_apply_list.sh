#!/bin/bash
# launch list of ONE preconditioner application (cfg2), plan replayed from a plain run
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export MGRX_GRAPHS=0
rm -f gpurun_out/plan_ap.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_ap.txt timeout 300 python tools/ncu_probe.py cfg2 precond.inexact > gpurun_out/ap_plain.log 2>&1
echo plain rc=$?
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_ap.txt timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/ap_launches.csv python tools/ncu_probe.py cfg2 precond.inexact > gpurun_out/ap_ncu.log 2>&1
echo rc=$?
