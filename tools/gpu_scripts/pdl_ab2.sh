#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for xt in 0 1; do for m in 0 2 0 2; do
  L=$PWD/paper_2101_11649_b200/libmgrx_p$m.so
  [ $m = 0 ] && L=$PWD/paper_2101_11649_b200/libmgrx.so
  MGRX_SPMV_XT=$xt MGRX_LIB=$L timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_pdl.log 2>&1
  echo "xt $xt mode $m $(grep -h '^{' gpurun_out/bench_pdl.log | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["iterations_per_solve"], d["roofline"]["kernels"]["precond.inexact"]["avg_ms"])')"
done; done
MGRX_LIB=$PWD/paper_2101_11649_b200/libmgrx_p2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -n 1
