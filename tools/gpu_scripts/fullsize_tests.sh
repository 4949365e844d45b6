#!/bin/bash
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 3000 python -m pytest tests/test_gpu_fullsize.py -q -x --durations=10 > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
tail -n 25 gpurun_out/pytest_full.log
