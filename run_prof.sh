#!/bin/bash
# ncu --set full of the level-1 / level-2 AMG residual SpMV (cfg2), staged
# choices replayed from a plain run
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
rm -f gpurun_out/plan_probe.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_probe.txt python tools/probe_spmv.py amg.1.resid amg.2.resid spmv.A > gpurun_out/probe_plain.log 2>&1
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_probe.txt ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spmv -c 3 -o gpurun_out/amg12_full -f python tools/probe_spmv.py amg.1.resid amg.2.resid spmv.A > gpurun_out/ncu_amg12.log 2>&1
echo done
