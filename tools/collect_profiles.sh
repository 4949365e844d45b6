#!/bin/bash
# Copy the evidence of tools/gpu_scripts/final_round.sh from gpurun_out/ into
# profiles/r01/ (bench JSON lines, launch lists, launch shares, SpMV plans,
# step timeline).
set -e
cd "$(dirname "$0")/.."
O=gpurun_out
P=profiles/r01
line() { grep -h '^{' "$1" | tail -n 1; }
line $O/bench.log > $P/bench_cfg2.json
line $O/bench_ref.log > $P/bench_cfg2_reference.json
for c in cfg3 cfg4 cfg5; do line $O/bench_$c.log > $P/bench_$c.json; done
cp $O/launches_cfg2.csv $P/launches_bench_timed.csv
cp $O/launches_cfg3.csv $P/launches_cfg3_timed.csv
cp $O/launches_cfg4.csv $P/launches_cfg4_timed.csv
for c in cfg2 cfg3 cfg4; do cp $O/plan_$c.txt $P/spmv_plan_$c.txt; done
hdr() {
  echo "launches in one timed $1 solve ($2; ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none,"
  echo "serialised, cold cache; SpMV plan choices replayed from spmv_plan_$1.txt); ns."
}
{ hdr cfg2 mfd_mgr_pi_c1_l1j; python tools/launch_stats.py $P/launches_bench_timed.csv; } > $P/launch_shares.txt
{ hdr cfg3 comp_mgr_l1j; python tools/launch_stats.py $P/launches_cfg3_timed.csv; } > $P/launch_shares_cfg3.txt
{ hdr cfg4 frac_mgr_u_l1j; python tools/launch_stats.py $P/launches_cfg4_timed.csv; } > $P/launch_shares_cfg4.txt
{
  echo "GMRES_PROF (MGRX_GMRES_PROF=1, cfg2, per solve, ms; 'gap' = host time from a step's D2H to the next step's first kernel, plus the restart work between cycles)"
  grep -h GMRES_PROF $O/bench_steps.log
} > $P/gmres_step_timeline.txt
echo collected
