"""Summarise ptxas -v output: registers / spill bytes / stack per kernel (demangled-ish)."""
import re
import sys

cur = None
rows = {}
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["stack"], rows[cur]["st"], rows[cur]["ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for k, v in rows.items():
    if pat in k:
        name = re.sub(r"_ZN3ssb\d+_GLOBAL__N__\w+?_sart_cu_\w+?\d\d", "", k)
        print(f"{v.get('regs','?'):>4} regs  spill st/ld {v.get('st',0)}/{v.get('ld',0)}  {name[:90]}")
