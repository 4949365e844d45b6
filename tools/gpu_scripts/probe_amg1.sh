#!/bin/bash
# cfg2 AMG level-1/2 operator probes under alternative staged geometries, then
# one ncu --set full capture of the level-1 residual (plan replayed from a
# plain run: ncu distorts the setup timing)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
P="amg.1.resid amg.1.pre amg.2.resid amg.2.pre"
rm -f gpurun_out/plan_amg1.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_amg1.txt timeout 300 python tools/probe_spmv.py $P > gpurun_out/probe_default.log 2>&1
MGRX_SPMV_GEOM=1 timeout 300 python tools/probe_spmv.py $P > gpurun_out/probe_geom1.log 2>&1
MGRX_SPMV_CTAS=3 timeout 300 python tools/probe_spmv.py $P > gpurun_out/probe_ctas3.log 2>&1
MGRX_SPMV_CTAS=2 timeout 300 python tools/probe_spmv.py $P > gpurun_out/probe_ctas2.log 2>&1
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_amg1.txt timeout 600 ncu --set full --clock-control none --import-source on \
  --profile-from-start off -k regex:k_spmv -c 1 -o gpurun_out/amg1_resid -f \
  python tools/probe_spmv.py amg.1.resid > gpurun_out/ncu_amg1.log 2>&1
grep -h avg20 gpurun_out/probe_*.log
