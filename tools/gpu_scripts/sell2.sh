#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in cfg2 cfg4; do
MGRX_VERBOSE=1 timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-variant 2>gpurun_out/sell2_err_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c ms', d['ms_per_step'], 'its', d['iterations_per_solve'], {k:(round(v.get('avg_ms',0)*1e3,1), round(v.get('GBps',0))) for k,v in d['roofline']['kernels'].items() if 'amg' in k or 'mgr' in k})"
grep -E "sell" gpurun_out/sell2_err_$c.log | head -20
done
