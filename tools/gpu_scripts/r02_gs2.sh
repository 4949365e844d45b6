#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gauss_seidel_block" > gpurun_out/pytest_gs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gs.log
for b in 12288 4096 2048; do MGRX_GS_BLK_ROWS=$b timeout 600 python tools/gpu_scripts/gs_check.py; done > gpurun_out/gs_check2.log 2>&1
tail -3 gpurun_out/pytest_gs.log; cat gpurun_out/gs_check2.log
