#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
tail -n 40 gpurun_out/pytest_shard.log
