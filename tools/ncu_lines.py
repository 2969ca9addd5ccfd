"""Aggregate ncu warp-stall samples per CUDA source line from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kfilter = sys.argv[3] if len(sys.argv) > 3 else None  # substring of the function name
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
agg = defaultdict(float)
src = {}
fname = "?"
func = ""
hdr = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= si:
        continue
    if kfilter and kfilter not in func:
        continue
    if r[0]:
        line = (fname, r[0])
        src[line] = r[1]
    try:
        agg[line] += float(r[si] or 0)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / tot * 100:5.1f}%  {k[0]}:{k[1]:>5}  {src.get(k, '')[:100].strip()}")
print("total samples", tot)
