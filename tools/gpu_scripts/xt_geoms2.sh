#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "xwindow or pattern or spmv" 2>&1 | tail -n 1
for g in ${GEOMS:-0 1 2 3}; do
echo "== geom $g warm"; MGRX_SPMV_XT_GEOM=$g MGRX_SPMV_XT=2 timeout 600 python tools/probe_spmv.py amg.1.resid amg.1.pre amg.0.resid amg.2.resid spmv.A 2>&1 | grep avg20
echo "== geom $g cold"; MGRX_PROBE_FLUSH=1 MGRX_SPMV_XT_GEOM=$g MGRX_SPMV_XT=2 timeout 600 python tools/probe_spmv.py amg.1.resid amg.1.pre amg.0.resid amg.2.resid spmv.A 2>&1 | grep avg20
done
