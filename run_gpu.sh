#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --steps 3 --warmup 3 --strategy mfd_mgr_pi_c1_l1j --no-cpu-baseline > gpurun_out/bench_l1j.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_l1j.log
timeout 900 python bench.py --steps 2 --warmup 3 --strategy mfd_mgr_pi --no-cpu-baseline > gpurun_out/bench_c8.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c8.log
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
