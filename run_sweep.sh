#!/bin/bash
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 600 python tools/probe_gs_levels.py 2>&1 | grep -v spmv_prepare | grep "pre\|post" | tail -12
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms', round(d['ms_per_step'],2), 'variant', {k:(round(v['ms_per_step'],1), v['iterations_per_solve']) for k,v in d['variants'].items()})
"
