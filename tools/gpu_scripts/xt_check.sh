#!/bin/bash
# pattern-coded / x-window SpMV: parity tests, then cfg2 A/B (same box)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pattern_coded or xwindow or spmv" > gpurun_out/pytest_xt.log 2>&1; echo "rc=$? $(tail -n 1 gpurun_out/pytest_xt.log)"
run() { # name, env...
  local name=$1; shift
  env "$@" MGRX_VERBOSE=1 timeout 600 python bench.py --config ${CFG:-cfg2} --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_$name.log 2> gpurun_out/bench_$name.err
  echo "$name $(grep -h '^{' gpurun_out/bench_$name.log | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["iterations_per_solve"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["roofline"]["kernels"].items() if "avg_ms" in v and ("amg" in k or "spmv" in k or "mgr" in k)})')"
}
run both A=1
run nopat MGRX_SPMV_PAT=0
run noxt MGRX_SPMV_XT=0
run none MGRX_SPMV_XT=0 MGRX_SPMV_PAT=0
grep -h "xtile\|staged_pat" gpurun_out/bench_both.err | sort | uniq -c | head -40
