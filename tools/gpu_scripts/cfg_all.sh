#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_xt.log 2>&1; echo "rc=$? $(tail -n 1 gpurun_out/pytest_xt.log)"
for c in ${CFGS:-cfg4 cfg2 cfg3 cfg5}; do
MGRX_VERBOSE=1 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant 2> gpurun_out/err_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d[\"ms_per_step\"], d[\"setup_s\"], d[\"iterations_per_solve\"], d['roofline']['kernels'].get('precond.inexact',{}).get('avg_ms'), d['solve_roofline'].get('frac'))"
grep -h "tune_spmv" gpurun_out/err_$c.log | cut -c1-120
done
