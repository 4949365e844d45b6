#!/bin/bash
# after the two-rows-per-thread short-row kernel / two-element jacobi0: probes + bitwise tests
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/probe_cold.py > gpurun_out/tpr_probe.log 2>&1
grep "solve_ms\|probe" gpurun_out/tpr_probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/tpr_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tpr_pytest.log
for c in cfg3 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-variant > gpurun_out/tpr_bench_$c.log 2>&1; grep '^{' gpurun_out/tpr_bench_$c.log | tail -1 | cut -c1-200; done
