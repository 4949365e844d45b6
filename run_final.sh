#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
rm -f gpurun_out/spmv_plan.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/spmv_plan.txt python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_prof_plain.log 2>&1 && \
MGRX_SPMV_PLAN_FILE=gpurun_out/spmv_plan.txt MGRX_PROFILE_TIMED=1 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/ncu_bench.log 2>&1
python tools/probe_spmv.py spmv.A > gpurun_out/probe_spmv_plain.log 2>&1 && \
MGRX_SPMV_PLAN_FILE=gpurun_out/spmv_plan.txt ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spmv -c 1 -o gpurun_out/spmv_full python tools/probe_spmv.py spmv.A > gpurun_out/ncu_spmv.log 2>&1
python tools/probe_spmv.py arnoldi.15 > gpurun_out/probe_arnoldi_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_arnoldi -c 1 -o gpurun_out/arnoldi_full python tools/probe_spmv.py arnoldi.15 > gpurun_out/ncu_arnoldi.log 2>&1
MGRX_GMRES_PROF=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_steps.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
