#!/usr/bin/env python3
"""Summarise an ncu report (raw page) and a launch-list CSV into profiles/.

  python tools/ncu_summary.py <report.ncu-rep> <out.json> [launches.csv]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__cycles_elapsed.avg.per_second",
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    header, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(header, units, r):
            if h in ("Kernel Name", "ID") or h in KEYS or any(h.startswith(k) for k in KEYS):
                d[h] = (v, u)
        res.append(d)
    return res


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r.get("Metric Unit")))
    agg = {}
    for name, v, unit in rows:
        key = name.split("(")[0]
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1.0)
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    total = sum(v[1] for v in agg.values()) or 1.0
    return {k: {"launches": c, "total_ms": t, "share": t / total} for k, (c, t) in
            sorted(agg.items(), key=lambda kv: -kv[1][1])}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    data = {"kernels": raw(rep)}
    if len(sys.argv) > 3:
        data["launch_list"] = launches(sys.argv[3])
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(data, indent=1)[:4000])


if __name__ == "__main__":
    main()
