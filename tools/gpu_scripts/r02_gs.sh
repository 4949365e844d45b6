#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gauss_seidel_block or cfg1_all or golden or solve_parity" > gpurun_out/pytest_gs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gs.log
for b in default 0 4096 8192; do
  if [ $b = default ]; then timeout 600 python tools/gpu_scripts/gs_check.py; else MGRX_GS_BLK_ROWS=$b timeout 600 python tools/gpu_scripts/gs_check.py; fi
done > gpurun_out/gs_check.log 2>&1
tail -5 gpurun_out/pytest_gs.log; cat gpurun_out/gs_check.log
