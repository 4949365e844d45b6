#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
MGRX_VERBOSE=1 timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gs.log 2>&1
MGRX_GS_MODE=lv timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gs_sf.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -k "bit_exact or solve_parity or cfg1" > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --strategy mfd_mgr_pi_c1_l1j --no-cpu-baseline > gpurun_out/bench_l1j.log 2>&1
python tools/profile_solve.py --strategy mfd_mgr_pi_c1_l1j --iters 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_l1j.csv python tools/profile_solve.py --strategy mfd_mgr_pi_c1_l1j --iters 3 > gpurun_out/ncu_l1j.log 2>&1
python tools/profile_solve.py --strategy mfd_mgr_pi_c1 --iters 2 > gpurun_out/prof_plain_gs.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_gs.csv python tools/profile_solve.py --strategy mfd_mgr_pi_c1 --iters 2 > gpurun_out/ncu_gs.log 2>&1
echo done
