#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --sharded --steps 3 --warmup 3 > gpurun_out/bench_sharded1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sharded1.log
CONFIGS="cfg2 cfg3 cfg4 cfg5" bash tools/gpu_scripts/r02_launches.sh > /dev/null 2>&1
tail -n 2 gpurun_out/bench_sharded1.log | cut -c1-1500
for c in cfg2 cfg3 cfg4 cfg5; do echo "== $c"; grep '^{' gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['iterations_per_solve'], d['value'], d['e2e']['value'], d['roofline']['kernel'], {k:(round(v.get('avg_ms',0)*1e3,1), round(v.get('GBps',0))) for k,v in d['roofline']['kernels'].items()})"; head -n 14 gpurun_out/shares_$c.txt; done
