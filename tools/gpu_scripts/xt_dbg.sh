#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for d in ${DBGS:-0 2 4 6 8 14}; do
echo "== MGRX_XT_DBG=$d flush"
MGRX_XT_DBG=$d MGRX_SPMV_XT_GEOM=${GEOM:-0} MGRX_SPMV_XT=2 MGRX_PROBE_FLUSH=1 timeout 600 python tools/probe_spmv.py amg.1.resid amg.0.resid 2>&1 | grep avg20
echo "== MGRX_XT_DBG=$d warm"
MGRX_XT_DBG=$d MGRX_SPMV_XT_GEOM=${GEOM:-0} MGRX_SPMV_XT=2 timeout 600 python tools/probe_spmv.py amg.1.resid amg.0.resid 2>&1 | grep avg20
done
