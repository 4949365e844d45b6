#!/bin/bash
mkdir -p gpurun_out
TAG=small python tools/probe_gs.py > gpurun_out/probe_trace.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -k "bit_exact or solve_parity or apply or cfg1 or alternative or edge" >> gpurun_out/probe_trace.log 2>&1
echo done
