#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pattern_coded or xwindow or spmv or solve_parity" > gpurun_out/pytest_xt.log 2>&1; echo "rc=$? $(tail -n 1 gpurun_out/pytest_xt.log)"
run() { # name cfg env...
  local name=$1; local cfg=$2; shift; shift
  env "$@" MGRX_VERBOSE=1 MGRX_PROBE_FLUSH=1 timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_$name.log 2> gpurun_out/bench_$name.err
  echo "$name $(grep -h '^{' gpurun_out/bench_$name.log | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["iterations_per_solve"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["roofline"]["kernels"].items() if "avg_ms" in v and ("amg" in k or "spmv" in k or "mgr" in k or "precond" in k)})')"
}
run xt_cfg2 cfg2 A=1
run xtg0_cfg2 cfg2 MGRX_SPMV_XT_GEOM=0
run xtg1_cfg2 cfg2 MGRX_SPMV_XT_GEOM=1
run noxt_cfg2 cfg2 MGRX_SPMV_XT=0
grep -h "xtile" gpurun_out/bench_xt_cfg2.err | head -60
