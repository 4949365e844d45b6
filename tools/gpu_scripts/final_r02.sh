#!/bin/bash
# End-of-round-2 evidence: GPU suite, smoke, bench lines (cfg2 full + reference arm,
# cfg3-5, sharded N=1), launch lists cfg2-4, ncu --set full of the roofline kernels.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_cfg2.log 2>&1
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
for c in cfg3 cfg4 cfg5; do timeout 1200 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
timeout 900 python bench.py --sharded --steps 3 --warmup 3 > gpurun_out/bench_sharded1.log 2>&1
CONFIGS="cfg2 cfg3 cfg4" bash tools/gpu_scripts/launch_list_cfg.sh > gpurun_out/launch_lists.log 2>&1
CFG=cfg2 PROBES="spmv.A cgs2dots.15 cgs2upd.15 amg.1.resid amg.0.pre amg.1.pre amg.2.resid" bash tools/gpu_scripts/r02_ncu.sh > gpurun_out/ncu_all.log 2>&1
CFG=cfg4 PROBES="mgr.0.frelax.amg.0.resid mgr.0.frelax.amg.1.resid" bash tools/gpu_scripts/r02_ncu.sh > gpurun_out/ncu_cfg4.log 2>&1
rm -f gpurun_out/*.ncu-rep
tail -4 gpurun_out/pytest_gpu_all.log; tail -2 gpurun_out/smoke.log
for f in bench_cfg2 bench_ref bench_cfg3 bench_cfg4 bench_cfg5 bench_sharded1; do grep '^{' gpurun_out/$f.log | tail -1 | cut -c1-300; done
