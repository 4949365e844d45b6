#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "team_sum" > gpurun_out/vec_tests.log 2>&1; echo "rc=$?" >> gpurun_out/vec_tests.log
tail -5 gpurun_out/vec_tests.log
MGRX_VERBOSE=1 timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/vec_cfg4.log 2> gpurun_out/vec_cfg4.err
grep "bsr(3)" gpurun_out/vec_cfg4.err | head
grep '^{' gpurun_out/vec_cfg4.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['iterations_per_solve'], d['solve_roofline']['frac'], d['solve_roofline'].get('precond_apply'), d['setup_s'])"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "cfg4" > gpurun_out/vec_fullsize.log 2>&1; tail -3 gpurun_out/vec_fullsize.log
