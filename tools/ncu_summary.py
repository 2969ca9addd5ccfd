"""Summarise ncu reports (``--set full`` captures and ``gpu__time_duration`` launch lists) as markdown.

    python tools/ncu_summary.py full  <report.ncu-rep> [--bytes-per-launch KERNEL=BYTES ...]
    python tools/ncu_summary.py launches <launches.csv>
    python tools/ncu_summary.py traffic <report.ncu-rep> <workload/sampler> [sweeps=S]
        -> merges {"<workload/sampler>/<kernel>": {"bytes": dram read+write of its first captured
           launch[, "sweeps": S]}} into profiles/traffic.json (bench.py's roofline "traffic")

Reads the report with ``ncu -i ... --page raw --csv`` (no GPU needed) and prints, per profiled
launch: duration, DRAM bytes read/written (the roofline ``traffic``), DRAM / SM throughput, pipe
utilisation, occupancy, registers and the top warp-stall reasons.  Used to write ``profiles/``.
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_size", "cluster"),
])


def _raw(report: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def _to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v) * scale


def full(report: str, bpl: dict) -> str:
    hdr, units, rows = _raw(report)
    ix = {h: i for i, h in enumerate(hdr)}
    lines = [f"### `{report}`", ""]
    for r in rows:
        name = r[ix["Kernel Name"]]
        lines.append(f"#### {name}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        dur_us = None
        traffic = 0.0
        for k, label in KEYS.items():
            if k not in ix:
                continue
            v, u = r[ix[k]], units[ix[k]]
            if k == "gpu__time_duration.sum":
                dur_us = float(v) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
                lines.append(f"| {label} | {dur_us:.2f} us |")
                continue
            if k.startswith("dram__bytes"):
                b = _to_bytes(v, u)
                traffic += b
                lines.append(f"| {label} | {b / 1e6:.3f} MB |")
                continue
            lines.append(f"| {label} | {v} {u} |")
        if dur_us:
            lines.append(f"| traffic (read+write) | {traffic / 1e6:.3f} MB = {traffic / dur_us / 1e3:.1f} GB/s |")
        for kname, b in bpl.items():
            if kname in name and dur_us:
                lines.append(f"| algorithmic bytes | {b / 1e6:.3f} MB = {b / dur_us / 1e3:.1f} GB/s "
                             f"(traffic/algorithmic = {traffic / b:.2f}) |")
        st = [(h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(r[ix[h]] or 0))
              for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
        st.sort(key=lambda t: -t[1])
        lines.append("| top stalls (warps per issue) | " + ", ".join(f"{n} {v:.2f}" for n, v in st[:5]) + " |")
        lines.append("")
    return "\n".join(lines)


def launches(path: str, only: str = "") -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        if only and not name.startswith(only):
            continue
        t = float(r[ix["Metric Value"]]) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ix["Metric Unit"]], 1.0)
        agg.setdefault(name, []).append(t)
    tot = sum(sum(v) for v in agg.values()) or 1.0
    lines = [f"### `{path}` (ncu, cold-cache, serialised; compare shares)", "",
             "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.2f} | {sum(v) / tot:.3f} |")
    return "\n".join(lines) + "\n"


def traffic(report: str, key: str, sweeps: int | None) -> str:
    import json
    import os
    hdr, units, rows = _raw(report)
    ix = {h: i for i, h in enumerate(hdr)}
    tfile = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "traffic.json")
    data = json.load(open(tfile)) if os.path.exists(tfile) else {}
    seen = set()
    for r in rows:
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        if name in seen:
            continue
        seen.add(name)
        b = sum(_to_bytes(r[ix[k]], units[ix[k]]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        ent = {"bytes": b}
        if sweeps and name in ("k_sweep_fused", "k_sweep_wide"):
            ent["sweeps"] = sweeps
        data[f"{key}/{name}"] = ent
    json.dump(data, open(tfile, "w"), indent=1, sort_keys=True)
    return json.dumps(data, indent=1, sort_keys=True)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "traffic":
        sw = [int(a.split("=")[1]) for a in sys.argv[4:] if a.startswith("sweeps=")]
        print(traffic(path, sys.argv[3], sw[0] if sw else None))
        sys.exit(0)
    bpl = {}
    for a in sys.argv[3:]:
        if "=" in a:
            k, v = a.split("=", 1)
            bpl[k] = float(v)
    if mode == "full":
        print(full(path, bpl))
    else:
        print(launches(path, sys.argv[3] if len(sys.argv) > 3 else ""))
