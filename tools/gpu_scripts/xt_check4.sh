#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_xt.log 2>&1; echo "rc=$? $(tail -n 1 gpurun_out/pytest_xt.log)"
for d in 0 2; do for g in 0 1 2; do echo "== dbg $d geom $g warm"; MGRX_XT_DBG=$d MGRX_SPMV_XT_GEOM=$g MGRX_SPMV_XT=2 timeout 600 python tools/probe_spmv.py amg.1.resid amg.0.resid 2>&1 | grep avg20; done; done
echo "== no xt warm"; MGRX_SPMV_XT=0 timeout 600 python tools/probe_spmv.py amg.1.resid amg.0.resid amg.0.pre spmv.A mgr.0.rres 2>&1 | grep avg20
run() { # name cfg env...
  local name=$1; local cfg=$2; shift; shift
  env "$@" MGRX_VERBOSE=1 timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/bench_$name.log 2> gpurun_out/bench_$name.err
  echo "$name $(grep -h '^{' gpurun_out/bench_$name.log | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["iterations_per_solve"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["roofline"]["kernels"].items() if "avg_ms" in v and ("amg" in k or "spmv" in k or "mgr" in k or "precond" in k)})')"
}
run xt_cfg2 cfg2 A=1
run noxt_cfg2 cfg2 MGRX_SPMV_XT=0
grep -h "xtile" gpurun_out/bench_xt_cfg2.err | grep -- "->" | head -60
