#!/bin/bash
mkdir -p gpurun_out
MGRX_GS_MODE=sf python tools/profile_solve.py --strategy mfd_mgr_pi_c1 --iters 1 > gpurun_out/prof_plain_gs.log 2>&1 && \
MGRX_GS_MODE=sf ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_gs -c 4 -o gpurun_out/gs_full python tools/profile_solve.py --strategy mfd_mgr_pi_c1 --iters 1 > gpurun_out/ncu_gs_full.log 2>&1
echo rc=$?
