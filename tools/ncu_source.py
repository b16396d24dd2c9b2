"""Per-instruction stall attribution from an ncu report (source page, SASS).  Usage: ncu_source.py REP [N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
ex = h.index("Instructions Executed")
tot = sum(int(r[si]) for r in data if r[si].isdigit()) or 1
c = Counter()
for r in data:
    if r[si].isdigit():
        toks = r[src].split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        c[op.split(".")[0]] += int(r[si])
print("samples", tot)
print("  " + ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in c.most_common(16)))
for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:n]:
    print(f"{r[si]:>6} {r[ex]:>10}  {r[0][-5:]}  {r[src][:90]}")
