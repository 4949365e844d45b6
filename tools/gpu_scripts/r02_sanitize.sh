#!/bin/bash
# compute-sanitizer over the small cases (each tool in its own process)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
MGRX_ARNOLDI_SELFXCHG=1 timeout 900 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py small > gpurun_out/san_memcheck_selfxchg.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_selfxchg.log
MGRX_GS_BLK_ROWS=4096 MGRX_GS_BLK_FORCE=1 MGRX_SPMV_BSR=2 MGRX_SPMV_SELL=2 timeout 1500 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_memcheck_forced.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_forced.log
timeout 2400 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py small > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log
timeout 3000 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python tools/sanitize_cases.py small > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
for f in gpurun_out/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|sanitize cases ok" $f | tail -4; done
