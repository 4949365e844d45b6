#!/bin/bash
# A/B: x-window kernel on / off, cold and warm probes + whole solve
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in default:MGRX_NONE=1 xt0:MGRX_SPMV_XT=0 noinsitu:MGRX_TUNE_INSITU=0 default2:MGRX_NONE=1; do
  tag=${v%%:*}; kv=${v#*:}
  env $kv timeout 300 python tools/probe_cold.py > gpurun_out/xtab_$tag.log 2>&1
  echo "== $tag ($kv)"; grep "solve_ms\|probe" gpurun_out/xtab_$tag.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "spmv or xtile or window or staged or tail or determinism" > gpurun_out/xtab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/xtab_pytest.log
