#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "team_sum or corrupt_transfer" > gpurun_out/vec_tests.log 2>&1; echo "rc=$?" >> gpurun_out/vec_tests.log
timeout 2000 python -m pytest tests/test_gpu_fullsize.py -m gpu -q > gpurun_out/vec_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/vec_fullsize.log
for c in cfg4 cfg2 cfg3 cfg5; do
  MGRX_VERBOSE=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/vec_$c.log 2> gpurun_out/vec_$c.err
done
tail -5 gpurun_out/vec_tests.log; tail -5 gpurun_out/vec_fullsize.log
for c in cfg4 cfg2 cfg3 cfg5; do echo $c; grep '^{' gpurun_out/vec_$c.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['iterations_per_solve'], d['solve_roofline']['frac'], d['solve_roofline'].get('precond_apply'))"; done
