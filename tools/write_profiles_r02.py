"""Copy the evidence of tools/gpu_round2.sh (gpurun_out/r02/) into profiles/ and regenerate profiles/r02_ncu.md:
bench lines, the reference arm, per-CTA critical-path phases, sensitivity experiments, the ncu --set full summary of
k_sweep_wide (+ its DRAM traffic into profiles/traffic.json), the top source lines by stall samples, the launch list."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O = os.path.join(ROOT, "gpurun_out", "r02")
P = os.path.join(ROOT, "profiles")


def run(*cmd):
    return subprocess.run([sys.executable, *cmd], capture_output=True, text=True, cwd=ROOT).stdout


def clean(path):
    return "".join(line for line in open(path) if "Warning" not in line and "nanmean" not in line)


def main():
    for src, dst in [("bench_c4.json", "r02_bench_c4.json"), ("bench_c2.json", "r02_bench_c2.json"),
                     ("bench_c3.json", "r02_bench_c3.json"), ("bench_ref.json", "r02_bench_reference.json"),
                     ("bench_c5_slab8.json", "r02_bench_c5_slab8.json"), ("launches_c4.csv", "r02_launches_c4.csv")]:
        shutil.copy(os.path.join(O, src), os.path.join(P, dst))
    open(os.path.join(P, "r02_cta_c4.txt"), "w").write(clean(os.path.join(O, "cta_c4.txt")))
    open(os.path.join(P, "r02_sensitivity_c4.txt"), "w").write(clean(os.path.join(O, "sensitivity_c4.txt")))
    rep = os.path.join(O, "prof_c4.ncu-rep")
    run("tools/ncu_summary.py", "traffic", rep, "C4/leverage", "sweeps=2")
    full = run("tools/ncu_summary.py", "full", rep, "k_sweep_wide=196608000")
    stalls = run("tools/ncu_stalls.py", rep, "sweep_wide.cuh", "1", "2000")
    stalls = "\n".join(sorted(stalls.splitlines()[:-1], key=lambda l: -float(l.split()[1]) if len(l.split()) > 1 else 0)[:25])
    launch = run("tools/ncu_summary.py", "launches", os.path.join(P, "r02_launches_c4.csv"), "cps::")
    d4, d2, d3, dr, d5 = (json.load(open(os.path.join(P, f))) for f in
                          ("r02_bench_c4.json", "r02_bench_c2.json", "r02_bench_c3.json", "r02_bench_reference.json",
                           "r02_bench_c5_slab8.json"))
    tests = open(os.path.join(O, "pytest_gpu.log")).read().strip().splitlines()[-2]

    def line(d, name):
        r = d["roofline"] or {}
        ph = (d.get("phases") or {}).get("gather_roofline") or {}
        return (f"| {name} | {d['path']} | {d['value']:.4g} | {d['ms_per_step'] * 1e3:.1f} | {d['e2e']['value']:.4g} | "
                f"{r.get('kernel')} {r.get('achieved')} GB/s = {100 * (r.get('frac') or 0):.2f} % | "
                f"{(str(round(100 * ph['frac'], 1)) + ' %') if ph else '-'} | "
                f"{d['clocks']['sm_mhz']:.0f} MHz {d['clocks']['reasons']} |")

    out = f"""# Round 2 -- measured evidence (B200, this build)

Commands: `tools/gpu_round2.sh` (one gpurun call; this file: `tools/write_profiles_r02.py`): `pytest -m gpu` ({tests}),
`bench.py` (default: C4, N = 1), `bench.py --impl reference`, `bench.py --workload C2|C3`,
`bench.py --workload C5 --slab-of 8`, `tools/pw_cta.py C4`, `tools/pw_ablate.py C4`, the ncu launch list of
`bench.py --steps 5 --warmup 3` (`--metrics gpu__time_duration.sum --clock-control none`) and one `ncu --set full
--clock-control none --import-source on` capture of `k_sweep_wide` (one launch of 2 C4 sweeps, `tools/pw_ncu.py C4 2`,
`CPSGD_PW_NONCOOP=1`).  Files: `r02_bench_*.json`, `r02_launches_c4.csv`, `r02_cta_c4.txt`, `r02_sensitivity_c4.txt`.

## Bench lines (device clock, CUDA events; inputs larger than L2)

| workload | path | fibers/s | us / sweep | e2e fibers/s | roofline (whole launch) | gather phase | SM clock |
|---|---|---|---|---|---|---|---|
{line(d4, 'C4 (default)')}
{line(d2, 'C2')}
{line(d3, 'C3')}

Reference arm (the oracle, 1 core, bounded sample): {dr['value']} fibers/s; `cpu_baseline` of the C4 line:
{d4['cpu_baseline']['value']} fibers/s ({d4['cpu_baseline']['cores']} core).  C5, rank 0 of an 8-way slab split on one GPU
(exchanges excluded): {d5['ms_per_step'] * 1e3:.0f} us per sweep = {d5['value']:.4g} fibers/s of the global batch.

C4 `roofline`: one `k_sweep_wide` launch runs every phase of every SGD iteration of the timed sweeps, so its achieved
rate = the sampled fibers' bytes (3 x 4096 x 2000 x 4 B = 98.3 MB per sweep) / the launch time.  The DRAM traffic of
the captured launch (below) is ~1.06 x the algorithmic bytes: every fiber is read once; the step is latency-bound (the
serial chain of the method, R9), not bandwidth-bound.

## Per-CTA phase durations at C4 (`tools/pw_cta.py`; max over CTAs = the phase's share of the critical path)

```
{clean(os.path.join(O, 'cta_c4.txt'))}```

("S" includes the wait for the previous iteration's table units; the CTAs without table units reach it early, which
is what the S maximum shows.)

## Sensitivity experiments at C4 (`tools/pw_ablate.py`, timing only)

```
{clean(os.path.join(O, 'sensitivity_c4.txt'))}```

## ncu --set full: k_sweep_wide (C4, one launch of 2 sweeps)

{full}

Top source lines by stall samples (`tools/ncu_stalls.py`; `barrier` = CTAs waiting at the grid-wide syncs):

```
{stalls}
```

## Launch list (ncu, cold-cache, serialised)

{launch}
(`k_transpose` builds the mode-major copies at init; the e2e leg's host-buffer calls launch `k_take_compare`.)
"""
    open(os.path.join(P, "r02_ncu.md"), "w").write(out)
    print("profiles/r02_ncu.md written")


if __name__ == "__main__":
    main()
