#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "xwindow or pattern or spmv or solve_parity" > gpurun_out/pytest_xt.log 2>&1; echo "rc=$? $(tail -n 1 gpurun_out/pytest_xt.log)"
for two in 8 1000 4 16; do for g in 0 1; do echo "== two $two geom $g warm"; MGRX_XT_TWO=$two MGRX_SPMV_XT_GEOM=$g MGRX_SPMV_XT=2 timeout 600 python tools/probe_spmv.py amg.1.resid amg.0.resid amg.2.resid spmv.A 2>&1 | grep avg20; done; done
run() { # name cfg env...
  local name=$1; local cfg=$2; shift; shift
  env "$@" MGRX_VERBOSE=1 timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_$name.log 2> gpurun_out/bench_$name.err
  echo "$name $(grep -h '^{' gpurun_out/bench_$name.log | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["iterations_per_solve"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["roofline"]["kernels"].items() if "avg_ms" in v and ("amg" in k or "spmv" in k or "mgr" in k or "precond" in k)})')"
}
run xt_cfg2 cfg2 A=1
run xt1000_cfg2 cfg2 MGRX_XT_TWO=1000
grep -h "xtile" gpurun_out/bench_xt_cfg2.err | grep -- "->" | head -60
