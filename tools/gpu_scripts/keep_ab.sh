#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for k in 0 3000000; do
for c in cfg2 cfg3; do
  echo "keep_nnz=$k $c"
  MGRX_VEC_KEEP_NNZ=$k timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['solve_roofline'].get('precond_apply')['avg_ms'])"
done; done; done
