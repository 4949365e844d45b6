#!/bin/bash
# mgrx_solve_op parity tests + the default bench line with the cold-L2 family roofline
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "solve_op" > gpurun_out/solveop_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/solveop_pytest.log
tail -5 gpurun_out/solveop_pytest.log
timeout 1500 python bench.py --no-variant > gpurun_out/bench_cold.log 2>&1; echo "rc=$?"
grep '^{' gpurun_out/bench_cold.log | tail -1 | cut -c1-300
tail -3 gpurun_out/bench_cold.log | cut -c1-300
