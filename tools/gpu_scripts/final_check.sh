#!/bin/bash
# last check of HEAD: GPU suite, smoke, default bench (both arms)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 1200 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1
timeout 1500 python bench.py > gpurun_out/final_bench.log 2>&1
tail -3 gpurun_out/final_pytest.log; tail -2 gpurun_out/final_smoke.log
grep '^{' gpurun_out/final_bench_ref.log | tail -1 | cut -c1-250
grep '^{' gpurun_out/final_bench.log | tail -1 | cut -c1-400
