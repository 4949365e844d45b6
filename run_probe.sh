#!/bin/bash
mkdir -p gpurun_out
for pm in 0 1 2; do MGRX_GS_PUB=$pm TAG=pub$pm python tools/probe_gs.py; done > gpurun_out/probe_trace.log 2>&1
echo done
