#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in cfg2 cfg3 cfg5 cfg4; do
  MGRX_VERBOSE=1 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/is_$c.log 2> gpurun_out/is_$c.err
  echo $c; grep "tune_spmv.*team" gpurun_out/is_$c.err | head -8
  grep '^{' gpurun_out/is_$c.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['iterations_per_solve'], d['solve_roofline'].get('precond_apply')['avg_ms'], d['setup_s'])"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/parity.log 2>&1; tail -3 gpurun_out/parity.log
