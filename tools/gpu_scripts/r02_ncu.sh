#!/bin/bash
# ncu --set full of the roofline kernels (one probe launch each, profiler window)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CFG=${CFG:-cfg2}
for pr in ${PROBES:-spmv.A cgs2dots.15 cgs2upd.15 amg.1.resid}; do
  tag=$(echo $pr | tr '.' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -c 4 -f \
     -o gpurun_out/${CFG}_${tag} python tools/ncu_probe.py $CFG $pr > gpurun_out/ncu_${CFG}_${tag}.log 2>&1
  ncu -i gpurun_out/${CFG}_${tag}.ncu-rep --page raw --csv > gpurun_out/${CFG}_${tag}_raw.csv 2>/dev/null
done
ls -la gpurun_out/*.ncu-rep
