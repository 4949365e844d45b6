#!/bin/bash
# team-sum SpMV variants on the cfg4 / cfg2 hierarchies (per-matrix setup timings)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
cat > /tmp/vp.py <<'P'
import sys
sys.path.insert(0, '.')
import paper_2101_11649_b200 as mx
which = sys.argv[1]
if which == 'cfg4':
    P = mx.frac_problem(64, seed=20210131); t = mx.load_strategy('frac_mgr_u_l1j')
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t, P.unknown_map)
else:
    P = mx.mfd_problem(128, 128, 64, "layered", seed=20210129); t = mx.load_strategy('mfd_mgr_pi_c1_l1j')
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t)
P
for c in cfg4 cfg2; do
for v in "1 4" "2 4" "2 2" "2 8"; do
  set -- $v
  echo "== $c variant $1 grid x$2"
  MGRX_TUNE_INSITU=0 MGRX_VERBOSE=1 MGRX_VEC_VARIANT=$1 MGRX_VEC_GRID=$2 timeout 600 python /tmp/vp.py $c 2>&1 | grep "team-sum" | awk '!seen[$0]++' | cut -c1-200
done
done > gpurun_out/vec_probe.log 2>&1
cat gpurun_out/vec_probe.log
