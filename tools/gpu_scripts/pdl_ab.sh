#!/bin/bash
# A/B of the PDL modes (MGRX_PDL_MODE builds libmgrx_p<m>.so): L1 visibility
# test of griddepcontrol.wait, parity subset and cfg2 bench per mode.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pdl_l1_test tools/pdl_l1_test.cu && /tmp/pdl_l1_test > gpurun_out/pdl_l1_test.log 2>&1
cat gpurun_out/pdl_l1_test.log
for m in ${MODES:-0 7 3 6 1}; do
  L=$PWD/paper_2101_11649_b200/libmgrx_p$m.so
  [ $m = 0 ] && L=$PWD/paper_2101_11649_b200/libmgrx.so
  [ -f $L ] || continue
  MGRX_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_p$m.log 2>&1; echo "mode $m parity rc=$? $(tail -n 1 gpurun_out/pytest_p$m.log)"
  for c in cfg2 ${CFGS}; do
  MGRX_LIB=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_p${m}_$c.log 2>&1
  echo "mode $m $c $(grep -h '^{' gpurun_out/bench_p${m}_$c.log | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["iterations_per_solve"])')"
  done
done
