#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python tools/gpu_scripts/ls_check.py > gpurun_out/ls_check.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cgs2" > gpurun_out/pytest_cgs2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cgs2.log
cat gpurun_out/ls_check.log; tail -3 gpurun_out/pytest_cgs2.log
