#!/bin/bash
# team-sum SpMV: tests + quick bench lines of cfg2 / cfg4 / cfg3 with and without it
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "team_sum or corrupt_transfer or cgs2 or solve_entry" > gpurun_out/vec_tests.log 2>&1; echo "rc=$?" >> gpurun_out/vec_tests.log
for c in cfg4 cfg2 cfg3; do
  MGRX_VERBOSE=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/vec_$c.log 2> gpurun_out/vec_$c.err
  MGRX_SPMV_VEC=0 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/novec_$c.log 2>/dev/null
done
tail -3 gpurun_out/vec_tests.log
for c in cfg4 cfg2 cfg3; do for v in vec novec; do echo $v $c; grep '^{' gpurun_out/${v}_$c.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['iterations_per_solve'], d['solve_roofline']['frac'], d['solve_roofline'].get('precond_apply'))"; done; done
grep "team-sum" gpurun_out/vec_cfg4.err | head -40
grep "team-sum" gpurun_out/vec_cfg2.err | head -40
