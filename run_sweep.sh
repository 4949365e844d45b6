#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for c in cfg4; do for e in X=0 MGRX_SPMV_WSPEC=2 MGRX_SPMV_WSPEC=0; do echo "== $c $e"; env $e timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variant 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms', round(d['ms_per_step'],2), 'its', d['iterations_per_solve'], 'value %.3e'%d['value'], 'solvefrac', round(d['solve_roofline'].get('frac',0),3))
"; done; done > gpurun_out/bench_ws.log 2>&1
cat gpurun_out/bench_ws.log
