#!/bin/bash
# round-2 evidence: GPU suite (incl. full-size parity), smoke, bench lines
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_cfg2.log 2>&1
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
for c in cfg3 cfg4 cfg5; do timeout 1200 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
timeout 900 python bench.py --sharded --steps 3 --warmup 3 > gpurun_out/bench_sharded1.log 2>&1
tail -4 gpurun_out/pytest_gpu_all.log; tail -2 gpurun_out/smoke.log
for f in bench_cfg2 bench_ref bench_cfg3 bench_cfg4 bench_cfg5 bench_sharded1; do grep '^{' gpurun_out/$f.log | tail -1 | cut -c1-400; done
