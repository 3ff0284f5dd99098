"""Per-kernel share of device time from an ncu launch list.

usage: python tools/launch_summary.py launches_raw.csv out_launches.csv out_summary.txt "<command>"
(launches_raw.csv = stdout of `ncu --metrics gpu__time_duration.sum --csv --page raw <cmd>`;
non-CSV lines such as the program's own output are skipped.)
"""
import csv
import io
import re
import sys
from collections import defaultdict


def main():
    raw, out_csv, out_txt, cmd = sys.argv[1:5]
    lines = [l for l in open(raw) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr) and r[0] != ""]
    ik, it = hdr.index("Kernel Name"), hdr.index("gpu__time_duration.sum")
    data = [r for r in data if re.match(r"^[\d.,]+$", r[it])]
    unit_row = rows[1]
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(unit_row[it], 1.0)
    agg = defaultdict(lambda: [0, 0.0])
    with open(out_csv, "w") as f:
        f.write(f"# {cmd}\n# cold-cache, serialised per-launch times; compare shares, not absolutes\n")
        f.write("id,kernel,ns\n")
        for n, r in enumerate(data):
            ns = float(r[it].replace(",", "")) * scale
            name = r[ik].split("(")[0].strip()
            f.write(f'{n},"{name}",{ns:.0f}\n')
            agg[name][0] += 1
            agg[name][1] += ns
    total = sum(v[1] for v in agg.values()) or 1.0
    with open(out_txt, "w") as f:
        f.write("share  launches  avg_us  kernel\n")
        for name, (c, ns) in sorted(agg.items(), key=lambda t: -t[1][1]):
            f.write(f"{100 * ns / total:6.2f}% {c:7d} {ns / c / 1e3:9.2f}  {name}\n")
    print(open(out_txt).read()[:1500])


if __name__ == "__main__":
    main()
