#!/bin/bash
mkdir -p gpurun_out
TRACE=1 TAG=tmpl timeout 300 python tools/probe_arnoldi.py > gpurun_out/probe_arn.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/ba_1.json 2>gpurun_out/ba_1.err
echo done
