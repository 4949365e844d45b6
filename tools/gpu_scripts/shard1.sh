#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for e in "" "MGRX_SPMV_BSR=0" "MGRX_GRAPHS=0"; do
  echo "== $e"
  env $e timeout 900 python bench.py --sharded --steps 3 --warmup 3 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['iterations_per_solve'], d['gpu_launches'])"
done
MGRX_VERBOSE=1 timeout 900 python bench.py --sharded --steps 1 --warmup 1 2>&1 | grep -E "bsr|gs sweep" | head
