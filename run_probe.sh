#!/bin/bash
mkdir -p gpurun_out
python tools/probe_spmv.py mgs spmv.A > gpurun_out/probe_spmv_plain.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
import paper_2101_11649_b200 as mx
P=mx.mfd_problem(128,128,64,'layered',seed=20210129)
H=mx.Hierarchy(mx.Matrix(P.ptr,P.col,P.val),P.partition,mx.load_strategy('mfd_mgr_pi_c1_l1j'))
for nm in ['mgs','spmv.A']:
    ms,by=H.time_kernel(nm,reps=50); print(nm, ms, by/(ms*1e-3)/1e9)
" >> gpurun_out/probe_spmv_plain.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -k "solve_parity or cfg1" >> gpurun_out/probe_spmv_plain.log 2>&1
echo done
