"""Summarise an ncu --csv launch list: per-kernel count, time, DRAM bytes, L2 hit rate."""
import csv
import collections
import sys


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    return rows


def main(path):
    by = collections.OrderedDict()
    for r in load(path):
        key = (r["ID"], r["Kernel Name"])
        d = by.setdefault(key, {})
        v = r["Metric Value"].replace(",", "")
        try:
            d[r["Metric Name"]] = float(v)
        except ValueError:
            pass
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
    tot = 0.0
    for (i, name), d in by.items():
        short = name.split("(")[0][:60]
        t = d.get("gpu__time_duration.sum", 0.0)
        unit_ns = t  # ncu reports nsecond or usecond; normalised below
        a = agg[short]
        a[0] += 1
        a[1] += unit_ns
        a[2] += d.get("dram__bytes_read.sum", 0.0)
        a[3] += d.get("dram__bytes_write.sum", 0.0)
        a[4] += d.get("lts__t_sector_hit_rate.pct", 0.0)
        tot += unit_ns
    print(f"launches {len(by)}, sum time {tot:.1f} (ncu units)")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:18]:
        print(f"  {k:60s} n={a[0]:5d} t={a[1]:10.1f} {100*a[1]/tot:5.1f}%  avg={a[1]/a[0]:8.2f}"
              f"  rd/launch={a[2]/a[0]/1e6:7.2f}  wr/launch={a[3]/a[0]/1e6:7.2f}  l2hit={a[4]/a[0]:5.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
