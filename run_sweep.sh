#!/bin/bash
for lib in paper_2101_11649_b200/libmgrx_head.so paper_2101_11649_b200/libmgrx.so paper_2101_11649_b200/libmgrx_head.so paper_2101_11649_b200/libmgrx.so; do MGRX_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variant 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$lib', 'ms', round(d['ms_per_step'],2), 'arn', round(d['roofline']['kernels']['arnoldi.15']['avg_ms']*1e3,1))
"; done
