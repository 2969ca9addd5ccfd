"""Per-source-line stall breakdown from `ncu -i X --page source --csv --print-source cuda,sass`:
python tools/ncu_stalls.py report.ncu-rep file.cuh first_line last_line"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, fname, a, b = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
cur_file, line, hdr = None, None, None
agg = defaultdict(lambda: defaultdict(float))
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Name" or r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        try:
            line = int(r[0])
        except ValueError:
            continue
        src[(cur_file, line)] = r[1]
    if cur_file != fname or line is None or not (a <= line <= b):
        continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
            try:
                agg[line][h[6:]] += float(r[i] or 0)
            except ValueError:
                pass
tot = defaultdict(float)
for ln in sorted(agg):
    d = agg[ln]
    s = sum(d.values())
    if s < 1:
        continue
    top = sorted(d.items(), key=lambda kv: -kv[1])[:4]
    print(f"{ln:5d} {s:7.0f}  " + " ".join(f"{k}={v:.0f}" for k, v in top) + "   | " + src.get((fname, ln), "")[:70].strip())
    for k, v in d.items():
        tot[k] += v
print("total", {k: round(v) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]})
