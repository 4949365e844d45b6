#!/bin/bash
# profiling pass: ncu --set full on the level-1 AMG smoother SpMV and the MGR
# prolongation (cfg2), launch list of one timed cfg3 (comp_mgr_l1j) solve
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python tools/probe_spmv.py amg.1.pre mgr.0.prolong > gpurun_out/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spmv -c 2 -o gpurun_out/amg1_prolong_full -f python tools/probe_spmv.py amg.1.pre mgr.0.prolong > gpurun_out/ncu_amg1.log 2>&1
python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_cfg3_plain.log 2>&1 && \
MGRX_PROFILE_TIMED=1 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/ncu_cfg3.log 2>&1
echo done
