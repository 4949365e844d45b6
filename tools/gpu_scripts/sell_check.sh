#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "solve_paths_are_bit_exact" > gpurun_out/pytest_sell.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sell.log
for c in cfg2 cfg3 cfg5; do
for m in 1 0; do
echo "== $c MGRX_SPMV_SELL=$m"
MGRX_SPMV_SELL=$m MGRX_VERBOSE=1 timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-variant 2>gpurun_out/sell_err_${c}_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms', d['ms_per_step'], 'its', d['iterations_per_solve'], {k:(round(v.get('avg_ms',0)*1e3,1), round(v.get('GBps',0))) for k,v in d['roofline']['kernels'].items() if 'amg' in k or 'mgr' in k})"
grep -E "sell" gpurun_out/sell_err_${c}_$m.log | head -12
done; done > gpurun_out/sell_check.log 2>&1
tail -3 gpurun_out/pytest_sell.log; cat gpurun_out/sell_check.log
