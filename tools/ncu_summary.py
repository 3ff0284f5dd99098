"""Summarise an `ncu --set full` report (raw CSV page) per kernel.

usage: ncu -i rep.ncu-rep --page raw --csv > raw.csv
       python tools/ncu_summary.py raw.csv out_summary.json [traffic.json]

Writes the per-launch metrics the bench roofline cites (DRAM bytes, duration,
throughput, occupancy, issue activity, L1/L2 hit rates, top stall reasons);
with a third argument also (re)writes the `dram_bytes_per_launch` table that
bench.py reads, keyed by the kernel names ss_plan_describe reports.
"""
import csv
import json
import re
import sys
from collections import defaultdict

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l2_to_l1_sectors": "lts__t_sectors_srcunit_tex_op_read.sum",
    "grid": "launch__grid_size",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "msecond": 1e3,
         "nsecond": 1e-3}


def short(name):
    m = re.search(r"(sart_\w+<[^>]*>|\w+_kernel(<[^>]*>)?)", name)
    return m.group(1) if m else name


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(list)
    for d in data:
        rec = {}
        for key, m in METRICS.items():
            if m not in col:
                continue
            raw = d[col[m]].replace(",", "")
            try:
                v = float(raw)
            except ValueError:
                continue
            u = units[col[m]]
            if key.endswith("_bytes"):
                v *= SCALE.get(u, 1.0)
            if key == "duration_us":
                v *= SCALE.get(u, 1.0)
            rec[key] = v
        stalls = {}
        for h, i in col.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in h:
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        rec["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                                 for k, v in sorted(stalls.items(), key=lambda t: -t[1])[:4]}
        per[short(d[col["Kernel Name"]])].append(rec)
    out = {}
    for k, recs in per.items():
        avg = {}
        for key in METRICS:
            vals = [r[key] for r in recs if key in r]
            if vals:
                avg[key] = round(sum(vals) / len(vals), 3)
        avg["launches_captured"] = len(recs)
        avg["top_stalls_pct"] = recs[0]["top_stalls_pct"]
        if "dram_read_bytes" in avg:
            avg["dram_bytes_per_launch"] = avg["dram_read_bytes"] + avg.get("dram_write_bytes", 0)
        out[k] = avg
    json.dump(out, open(sys.argv[2], "w"), indent=1)
    if len(sys.argv) > 3:
        traffic = {k: {"dram_bytes_per_launch": v["dram_bytes_per_launch"],
                       "capture": sys.argv[2]}
                   for k, v in out.items() if "dram_bytes_per_launch" in v}
        json.dump(traffic, open(sys.argv[3], "w"), indent=1)
    for k, v in out.items():
        print(k, {x: v.get(x) for x in ("duration_us", "dram_bytes_per_launch", "dram_throughput_pct")})


if __name__ == "__main__":
    main()
