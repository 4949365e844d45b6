#!/bin/bash
export PYTHONUNBUFFERED=1
for k in -1 5 4 3 2 1 0; do
echo "cut $k: $(MGRX_VCYCLE_CUT=$k MGRX_TUNE_INSITU=${INSITU:-1} timeout 600 python tools/probe_spmv.py precond.inexact 2>&1 | grep avg20)"
done
