#!/bin/bash
# round 2, first low-sync check: build check, quick numbers, then the GPU suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python tools/gpu_scripts/ls_check.py > gpurun_out/ls_check.log 2>&1; echo "rc=$?" >> gpurun_out/ls_check.log
timeout 1200 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 30 gpurun_out/ls_check.log; tail -n 15 gpurun_out/pytest_gpu.log
