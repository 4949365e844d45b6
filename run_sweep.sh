#!/bin/bash
for c in cfg4 cfg2; do for e in X=0 MGRX_FUSE_J0=0 X=1 MGRX_FUSE_J0=0; do echo "== $c $e"; env $e timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-variant 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms', round(d['ms_per_step'],2), 'its', d['iterations_per_solve'], 'value %.3e'%d['value'])
"; done; done
