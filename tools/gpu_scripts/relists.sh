#!/bin/bash
# launch lists cfg2-4 again (plan replay fixed) + the DSMEM hand-off microbenchmark
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CONFIGS="cfg2 cfg3 cfg4" bash tools/gpu_scripts/launch_list_cfg.sh > gpurun_out/launch_lists.log 2>&1
head -12 gpurun_out/shares_cfg2.txt | cut -c1-140
timeout 60 ./tools/pingpong_dsmem > gpurun_out/pingpong_dsmem.txt 2>&1; cat gpurun_out/pingpong_dsmem.txt
