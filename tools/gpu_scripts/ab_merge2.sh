#!/bin/bash
# Same-box alternating A/B of the merged Arnoldi phase (cfg2 step timeline).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for r in 1 0 1 0; do
  MGRX_ARNOLDI_MERGE=$r MGRX_GMRES_PROF=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/abm_$r.log 2>&1
  echo "merge=$r $(grep -h GMRES_PROF gpurun_out/abm_$r.log | tail -n 1)"
  echo "merge=$r $(grep -h '^{' gpurun_out/abm_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernels"]["arnoldi.15"]["avg_ms"])')"
done
