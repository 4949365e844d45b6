#!/bin/bash
# ncu --set full of the x-window kernel with the Jacobi epilogue (amg.0.pre, all x-window plans on) and with the residual epilogue
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export MGRX_TUNE_INSITU=0
rm -f gpurun_out/plan_xj.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_xj.txt timeout 300 python tools/ncu_probe.py cfg2 amg.0.pre > gpurun_out/xj_plain.log 2>&1
echo plain rc=$?
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_xj.txt timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:k_spmv_xtile -s 3 -c 2 -o gpurun_out/xt_jac -f python tools/ncu_probe.py cfg2 amg.0.resid amg.0.pre > gpurun_out/xj_ncu.log 2>&1
echo ncu rc=$?
ncu -i gpurun_out/xt_jac.ncu-rep --page raw --csv > gpurun_out/xt_jac_raw.csv 2>/dev/null
ncu -i gpurun_out/xt_jac.ncu-rep --page source --csv --print-source sass > gpurun_out/xt_jac_source.csv 2>/dev/null
ls -la gpurun_out/xt_jac*
