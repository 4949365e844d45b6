#!/bin/bash
mkdir -p gpurun_out
TAG=kpoll8 python tools/probe_gs.py > gpurun_out/probe_trace.log 2>&1
for kp in 1 2; do MGRX_LIB=paper_2101_11649_b200/build/libmgrx_kpoll$kp.so TAG=kpoll$kp python tools/probe_gs.py >> gpurun_out/probe_trace.log 2>&1; done
echo done
