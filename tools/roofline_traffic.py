"""Summarise `ncu --set full` raw CSV exports of the roofline probes
(tools/gpu_scripts/r02_ncu.sh -> gpurun_out/<cfg>_<probe>_raw.csv) into
profiles/r02/roofline_traffic.json: per probe the kernel, DRAM bytes per launch
(dram__bytes_read.sum + dram__bytes_write.sum), duration, and the ratio to the
algorithmic bytes of the probe (taken from a bench line's roofline.kernels).

    python tools/roofline_traffic.py cfg2 profiles/r02/bench_cfg2.json gpurun_out profiles/r02/roofline_traffic.json \
        spmv.A cgs2dots.15 cgs2upd.15 amg.1.resid amg.0.pre
"""
import csv
import json
import os
import sys


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    u = unit.lower()
    return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)


def to_ms(v, unit):
    v = float(v.replace(",", ""))
    return v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit.lower(), 1e-3)


def main():
    cfg, bench_json, src, out = sys.argv[1:5]
    probes = sys.argv[5:]
    line = json.load(open(bench_json))
    kernels = {}
    for pr in probes:
        path = os.path.join(src, f"{cfg}_{pr.replace('.', '_')}_raw.csv")
        if not os.path.exists(path):
            continue
        rows = list(csv.reader(open(path)))
        hdr, units, vals = rows[0], rows[1], rows[2:]
        if not vals:
            continue
        idx = {h: i for i, h in enumerate(hdr)}
        v = vals[-1]  # the last profiled launch of the probe
        rd = to_bytes(v[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
        wr = to_bytes(v[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
        alg = line["roofline"]["kernels"].get(pr, {}).get("bytes")
        kernels[pr] = {
            "kernel": v[idx["Kernel Name"]][-90:],
            "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
            "algorithmic_bytes": alg,
            "traffic_over_algorithmic": (rd + wr) / alg if alg else None,
            "ncu_ms": to_ms(v[idx["gpu__time_duration.sum"]], units[idx["gpu__time_duration.sum"]]),
            "warps_active_pct": float(v[idx["smsp__warps_active.avg.pct_of_peak_sustained_active"]])
            if "smsp__warps_active.avg.pct_of_peak_sustained_active" in idx else None,
        }
    data = {}
    if os.path.exists(out):
        data = json.load(open(out))
    entry = data.get(cfg, {})
    entry.update({"config": cfg,
                  "source": "ncu --set full --clock-control none --import-source on, one probe launch in a profiler "
                            "window (tools/ncu_probe.py), cold L2 between replays",
                  "kernels": kernels})
    data[cfg] = entry
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(kernels, indent=1))


if __name__ == "__main__":
    main()
