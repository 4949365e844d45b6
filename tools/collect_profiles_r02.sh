#!/bin/bash
# Copy the evidence of tools/gpu_scripts/final_r02.sh from gpurun_out/ into
# profiles/r02/ (bench JSON lines, launch lists + shares, SpMV plans, the
# ncu --set full raw pages of the roofline probes and their traffic summary).
set -e
cd "$(dirname "$0")/.."
O=gpurun_out
P=profiles/r02
mkdir -p $P
line() { grep -h '^{' "$1" | tail -n 1; }
line $O/bench_cfg2.log > $P/bench_cfg2.json
line $O/bench_ref.log > $P/bench_cfg2_reference.json
for c in cfg3 cfg4 cfg5; do line $O/bench_$c.log > $P/bench_$c.json; done
[ -s $O/bench_sharded1.log ] && line $O/bench_sharded1.log > $P/bench_cfg2_sharded_n1.json
for c in cfg2 cfg3 cfg4; do
  [ -s $O/launches_$c.csv ] || continue
  cp $O/launches_$c.csv $P/launches_${c}_timed.csv
  cp $O/plan_$c.txt $P/spmv_plan_$c.txt
  {
    echo "launches in one timed $c solve (host-driven GMRES loop: ncu does not see inside the conditional-graph cycle;"
    echo "ncu --metrics gpu__time_duration.sum --clock-control none, serialised, cold cache; SpMV plan choices replayed"
    echo "from spmv_plan_$c.txt); ns."
    python tools/launch_stats.py $P/launches_${c}_timed.csv
  } > $P/launch_shares_$c.txt
done
for f in $O/cfg2_*_raw.csv $O/cfg4_*_raw.csv; do
  [ -s "$f" ] || continue
  b=$(basename "$f" _raw.csv)
  cp "$f" $P/ncu_${b}_full_raw.csv
done
python tools/roofline_traffic.py cfg2 $P/bench_cfg2.json $O $P/roofline_traffic.json \
  spmv.A cgs2dots.15 cgs2upd.15 amg.1.resid amg.0.pre amg.1.pre amg.2.resid
python tools/roofline_traffic.py cfg4 $P/bench_cfg4.json $O $P/roofline_traffic.json \
  mgr.0.frelax.amg.0.resid mgr.0.frelax.amg.1.resid
python - <<'PY'
import json, re
shares = {}
for line in open("profiles/r02/launch_shares_cfg2.txt"):
    m = re.match(r"\s+(?:void )?mgrx::<unnamed>::(\w+).*?t=\s*[\d.]+\s+([\d.]+)%", line)
    if m:
        shares[m.group(1)] = round(shares.get(m.group(1), 0.0) + float(m.group(2)) / 100.0, 4)
top = dict(sorted(shares.items(), key=lambda kv: -kv[1])[:6])
top["source"] = "profiles/r02/launch_shares_cfg2.txt"
d = json.load(open("profiles/r02/roofline_traffic.json"))
d["cfg2"]["launch_shares"] = top
json.dump(d, open("profiles/r02/roofline_traffic.json", "w"), indent=1)
print(top)
PY
tail -n 3 $O/pytest_gpu_all.log > $P/pytest_gpu_summary.txt
tail -n 3 $O/smoke.log >> $P/pytest_gpu_summary.txt
echo collected
