#!/bin/bash
# what the amg.1.pre / amg.1.post probes launch, and how long each launch takes cold (ncu launch list)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
rm -f gpurun_out/plan_a1.txt
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_a1.txt timeout 300 python tools/ncu_probe.py cfg2 amg.1.pre > gpurun_out/a1_plain.log 2>&1
MGRX_SPMV_PLAN_FILE=gpurun_out/plan_a1.txt timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/a1_launches.csv python tools/ncu_probe.py cfg2 amg.1.resid amg.1.pre amg.1.post amg.0.pre amg.2.pre > gpurun_out/a1_ncu.log 2>&1
echo rc=$?
grep -v "^==" gpurun_out/a1_launches.csv | cut -d, -f5,12- | head -60
