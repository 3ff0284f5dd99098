"""Run-length view of an ncu launch list (raw CSV page): which kernels repeat
back to back, and the per-kernel counts."""
import collections
import csv
import io
import re
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(io.StringIO("".join(lines))))
h = rows[0]
ik = h.index("Kernel Name")
seq = [re.sub(r"ssb::<unnamed>::", "", r[ik].split("(")[0])[:70] for r in rows[2:] if len(r) == len(h)]
print("launches", len(seq))
for k, n in collections.Counter(seq).most_common(8):
    print(f"{n:6d} {k}")
prev, n, runs = None, 0, []
for s in seq + [None]:
    if s == prev:
        n += 1
        continue
    if prev is not None and n > 1 and "sart" in prev:
        runs.append((len(runs), prev, n))
    prev, n = s, 1
print("repeated SART runs:", runs[:20])
