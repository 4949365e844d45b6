#!/bin/bash
mkdir -p gpurun_out
TAG=pipe python tools/probe_gs.py > gpurun_out/probe_trace.log 2>&1
MGRX_GS_MODE=sf TAG=sf python tools/probe_gs.py >> gpurun_out/probe_trace.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x >> gpurun_out/probe_trace.log 2>&1
echo done
