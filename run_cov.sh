#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "partition or block or dense_ideal or errors or setup_bit_exact or solve_parity" > gpurun_out/pytest_cov.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cov.log
tail -n 30 gpurun_out/pytest_cov.log
