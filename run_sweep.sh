#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_shard.py -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --sharded --steps 3 --warmup 2 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms', round(d['ms_per_step'],2), 'its', d['iterations_per_solve'], d['fused_sharded_arnoldi'])
"
