#!/bin/bash
mkdir -p gpurun_out
python tools/probe_spmv.py spmv.A amg.0.resid amg.0.pre mgr.0.prolong mgr.0.rres amg.1.resid amg.1.pre > gpurun_out/probe_spmv_plain.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -k "spmv or bit_exact or solve_parity" >> gpurun_out/probe_spmv_plain.log 2>&1
echo done
