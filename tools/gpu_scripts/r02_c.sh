#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
timeout 1500 python tools/shard_footprint.py --n 8 --out gpurun_out/shard_footprint.json > gpurun_out/footprint.log 2>&1; echo "rc=$?" >> gpurun_out/footprint.log
# launch list with the host-driven loop (ncu does not profile conditional-graph bodies)
rm -f gpurun_out/plan_cfg2.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_cfg2.txt timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_cfg2.log 2>&1
MGRX_GMRES_GRAPH=0 MGRX_SPMV_PLAN_FILE=gpurun_out/plan_cfg2.txt MGRX_PROFILE_TIMED=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_cfg2_host.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/ncu_cfg2.log 2>&1
python tools/launch_stats.py gpurun_out/launches_cfg2_host.csv > gpurun_out/shares_cfg2_host.txt 2>&1
MGRX_GMRES_GRAPH=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_cfg2_hostloop.log 2>&1
tail -3 gpurun_out/pytest_shard.log; tail -3 gpurun_out/footprint.log | cut -c1-1500; head -30 gpurun_out/shares_cfg2_host.txt
for f in bench_cfg2 bench_cfg2_hostloop; do grep '^{' gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['ms_per_step'], d['iterations_per_solve'], d['gpu_launches'])"; done
