#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bsr" > gpurun_out/pytest_bsr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bsr.log
for m in 0 1 2; do
echo "== MGRX_SPMV_BSR=$m"
MGRX_SPMV_BSR=$m MGRX_VERBOSE=1 timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline --no-variant 2>gpurun_out/bsr_err_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms', d['ms_per_step'], 'its', d['iterations_per_solve'], {k:(round(v.get('avg_ms',0)*1e3,1), round(v.get('GBps',0))) for k,v in d['roofline']['kernels'].items() if 'amg.0' in k or k=='spmv.A'})"
grep -E "bsr|csr" gpurun_out/bsr_err_$m.log | head -8
done > gpurun_out/bsr_check.log 2>&1
tail -3 gpurun_out/pytest_bsr.log; cat gpurun_out/bsr_check.log
