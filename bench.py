#!/usr/bin/env python
"""Benchmark of the importance-sampled SGD hot path (arXiv 2103.04081) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C2]
                    [--sampler leverage]

A "step" is one cyclic sweep: N_modes SGD iterations (one per mode), each running the whole hot
path -- table refresh (a1), sampling (a2, a3), SKR + fiber gather + contractions (a4-a6),
fixed/adaptive update (a7, a8) -- i.e. every SURVEY §8(a) row including the mode loop (a9).
metric = sampled fibers/s (whole job).  Default workload: BASELINE.json configs[3] (C4, 2000^3 fp32
= 32 GB, R = 50, B = 4096, adaptive step, leverage sampling) -- the largest configuration that fits one
GPU and the one whose fiber gather is HBM-bound; seeded synthetic data.

Multi-GPU (torchrun, one process per GPU): workloads that fit one GPU (C1-C4) run one independent
chain per GPU (different Philox seed, no collective; "scaling": "weak"); C5 runs slab-sharded
along the last mode with the NCCL allreduce / row broadcast inside the library ("strong").

--impl reference times the CPU oracle (oracle/liborc.so, single thread) on rank 0 on the same
workload, one SGD iteration (B fibers) per step (the paper publishes no GPU baseline; DESIGN.md
"Measurement").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "sampled fibers/s (cyclic sweeps of the importance-sampled SGD step)"
UNIT = "fibers/s"


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(cfg, device, seed_offset=0, slab=None):
    """seeded synthetic tensor + norm-matched U[0,1] init (synth)."""
    import torch

    if cfg.numel <= 200_000_000 and slab is None:
        X = synth.tensor(cfg)
        A0 = synth.init_factors(cfg, X)
        return torch.from_numpy(X).to(device), [torch.from_numpy(a).to(device) for a in A0], X, A0
    Xd, _, xnorm = synth.tensor_torch(cfg, device=device, slab=slab)
    A0 = synth.init_factors_torch(cfg, xnorm, device=device)
    return Xd, A0, None, None


def workload_str(cfg, sampler):
    """identical in both arms (the driver compares them)"""
    return (f"{cfg.name}: {'x'.join(map(str, cfg.dims))} {cfg.dtype}, R={cfg.rank}, B={cfg.batch}, {cfg.rule} step, "
            f"{sampler} sampling, cyclic mode order")


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu"] = line.split(":", 1)[1].strip()
                break
        info["mem_gb"] = round(os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2 ** 30, 1)
    except Exception:
        pass
    return info


def host_inputs(cfg):
    """the seeded tensor and initial factors on the host (numpy): the numpy recipe for tensors up to
    2e8 elements; larger ones are generated by the torch recipe on the GPU and copied to the host
    (fp32, read in place by the oracle's fp32 entry)"""
    if cfg.numel <= 200_000_000:
        X = synth.tensor(cfg)
        return X, synth.init_factors(cfg, X)
    import torch

    dev = torch.device("cuda:0")
    Xd, _, xn = synth.tensor_torch(cfg, device=dev)
    A0 = [a.cpu().numpy() for a in synth.init_factors_torch(cfg, xn, device=dev)]
    X = np.empty(cfg.numel, dtype=np.float32 if cfg.dtype == "f32" else np.float64)
    Xt = torch.from_numpy(X)
    chunk = 1 << 28
    for a in range(0, cfg.numel, chunk):
        Xt[a:a + chunk].copy_(Xd[a:a + chunk])
    del Xd
    torch.cuda.empty_cache()
    return X, A0


# ----------------------------------------------------------------------------------------------
def run_chains(args, cfg):
    """--chains K: K independent chains of the workload (same tensor, own factors
    and seeds) in ONE k_sweep_fused_multi launch per call, one cluster each; value = fibers/s summed
    over the chains.  Not the headline (that is one chain); a measure of the GPU's capacity."""
    import torch

    from paper_2103_04081_b200 import CPSGD

    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    Xd, Ad0, _, _ = make_inputs(cfg, dev)
    hs, keep = [], []
    for c in range(args.chains):
        Ad = [a.clone() for a in Ad0]
        h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=args.sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta,
                  seed=cfg.seed + 1000 * c, mode_major=not args.native_layout, fused_cluster=args.chain_cluster)
        hs.append(h)
        keep.append(Ad)
    CPSGD.sweep_multi(hs, args.warmup)
    for h in hs:
        h.sync()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        ev0.record()
        CPSGD.sweep_multi(hs, args.steps)
        for h in hs:
            h.sync()
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    N = cfg.order
    fibers = args.chains * N * cfg.batch * args.steps
    for h in hs:
        h.close()
    return {"metric": METRIC, "value": round(fibers / (ms / 1e3), 1), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if cfg.dtype == "f64" else "f32", "data": "synthetic (seeded; synth/ recipe)",
            "config": {"workload": f"{cfg.name}: {'x'.join(map(str, cfg.dims))} {cfg.dtype}, R={cfg.rank}, "
                                   f"B={cfg.batch}, {cfg.rule} step, {args.sampler} sampling, cyclic sweeps",
                       "chains": args.chains, "chain_cluster": args.chain_cluster, "step": f"one cyclic sweep of every chain ({N} SGD iterations x B "
                       f"fibers each), all chains in one k_sweep_fused_multi launch (one 16-CTA cluster each)",
                       "timing": "host-synchronised CUDA events around the call (all chains' streams)"},
            "clocks": clk.summary(), "gpu_launches": 1, "e2e": None}


def run_slab(args, cfg):
    """one rank's share of a slab-sharded run on ONE GPU -- rank 0 of the P-way split of the
    last mode (its slab of X, mode-major copies, an external-comm handle), timing the per-GPU sharded step (phases
    0-2 of every mode: the global batch's draws, the owned fibers' gather + contraction, the update, the table)
    with the exchanges left out.  value = the GLOBAL batch rate a P-GPU job would sustain if the exchanges were
    free (informational, not the driver's line)."""
    import torch

    from paper_2103_04081_b200 import CPSGD
    from paper_2103_04081_b200.parallel import slab_ranges

    P = args.slab_of
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    lo, hi = slab_ranges(cfg.dims[-1], P)[0]
    Xd, _, xn = synth.tensor_torch(cfg, device=dev, slab=(lo, hi))
    Ad = synth.init_factors_torch(cfg, xn, device=dev)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=args.sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta,
                  seed=cfg.seed, stream=stream, world_rank=0, world_size=P, slab=(lo, hi), external_comm=True,
                  fused=False)
    N = cfg.order

    def sweeps(k):
        for _ in range(k):
            for n in range(N):
                for ph in range(3):
                    h.step_phase(n, ph)

    sweeps(args.warmup)
    h.sync()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        ev0.record(stream)
        sweeps(args.steps)
        ev1.record(stream)
        stream.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = h.launches
    h.close()
    return {"metric": METRIC + " [one rank of a slab-sharded run, exchanges excluded]",
            "value": round(N * cfg.batch * args.steps / (ms / 1e3), 1), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic (seeded; synth/ recipe)",
            "config": {"workload": workload_str(cfg, args.sampler) + f"; rank 0 of {P} slabs [{lo}, {hi})",
                       "step": "one cyclic sweep of the rank's phases 0-2 (cp_sgd_step_phase), no exchange",
                       "slab_GB": round(Xd.numel() * 4 / 1e9, 2)},
            "clocks": clk.summary(), "gpu_launches": launches, "e2e": None}


def run_ours(args, cfg):
    import torch

    from paper_2103_04081_b200 import CPSGD

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.Stream(device=dev)
    # N > 1: C5 (256 GB) slab-sharded along the last mode (BASELINE configs[4]); every other workload ONE
    # chain on whole-tensor replicas with a batch split + allreduce of M (CP_FLAG_REPLICA; BASELINE
    # configs[3] "at 1/2/4/8 GPUs ... + allreduce", SURVEY 8(e) "C4 alternative"); --independent: one
    # unrelated chain per GPU (weak scaling)
    sharded = (cfg.name == "C5" and ws > 1)
    replica = (ws > 1 and not sharded and not args.independent)
    slab = None
    nccl_id = None
    if sharded:
        from paper_2103_04081_b200.parallel import slab_ranges

        slab = slab_ranges(cfg.dims[-1], ws)[rank]
    p2p = replica and args.exchange == "p2p"
    if sharded or (replica and not p2p):
        import torch.distributed as dist

        from paper_2103_04081_b200.cpsgd import nccl_unique_id

        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    Xd, Ad, Xh, A0h = make_inputs(cfg, dev, slab=slab)
    # the factors back to back in one device block (views): the host-buffer call moves them in one transfer each way
    flat = torch.empty(sum(a.numel() for a in Ad), dtype=Ad[0].dtype, device=dev)
    views, o = [], 0
    for a in Ad:
        v = flat[o:o + a.numel()].view(a.shape)
        v.copy_(a)
        views.append(v)
        o += a.numel()
    Ad = views
    torch.cuda.synchronize()
    one_chain = sharded or replica
    seed = cfg.seed if one_chain else cfg.seed + 1000 * rank  # independent chains: their own seeds
    t0 = time.time()
    with torch.cuda.stream(stream):
        h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=args.sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta,
                  seed=seed, stream=stream, world_rank=rank if one_chain else 0, world_size=ws if one_chain else 1,
                  nccl_id=nccl_id, slab=slab, mode_major=not args.native_layout, fused=args.path == "auto",
                  tc=not args.no_tc, replica=replica, p2p=p2p)
    if p2p:  # map every rank's exchange buffer (IPC handles all-gathered through torch.distributed)
        from paper_2103_04081_b200.parallel import p2p_connect

        p2p_connect(h)
    init_s = time.time() - t0
    h_path = h.path
    N = cfg.order
    fibers_per_step = sum(h.batch_max(n) for n in range(N)) if args.sampler.startswith("block") else N * cfg.batch

    def barrier():
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()

    # warm-up (captures the sweep graph)
    h.sweep(args.warmup)
    h.sync()
    # ---- timed region: K sweeps (graph replays) ----
    barrier()
    torch.cuda.synchronize()
    launches0 = h.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        h.sweep(args.steps)
        ev1.record(stream)
        stream.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = h.launches - launches0
    h.sync()
    if ws > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    total_fibers = fibers_per_step * args.steps * (1 if one_chain else ws)
    value = total_fibers / (ms / 1e3)

    # ---- per-kernel device durations (CUDA events on the launch stream, direct launches) ----
    h.profile(True)
    h.sweep(max(3, min(args.steps, 20)))
    prof = h.profile_read()
    h.profile(False)
    prof_sweeps = max(3, min(args.steps, 20))
    kern = {k: {"avg_us": 1e3 * t / c, "count": c, "share": 0.0} for k, (t, c) in prof.items()}
    tot = sum(t for t, c in prof.values()) or 1.0
    for k, (t, c) in prof.items():
        kern[k]["share"] = t / tot
    dominant = max(prof.items(), key=lambda kv: kv[1][0])[0] if prof else None

    peaks = load_peaks()
    esz = cfg.itemsize
    In_avg = sum(cfg.dims) / N
    if sharded:
        In_avg = (sum(cfg.dims[:-1]) + (slab[1] - slab[0])) / N
    # algorithmic bytes per k_gather launch: the sampled fibers (B_eff x I_n x sizeof); per the
    # sharded path only the locally owned part
    gather_bytes = (fibers_per_step / N) * In_avg * esz / (ws if replica else 1)  # replicas: this rank's chunks
    useful_gbs = value * (sum(cfg.dims) / N) * esz / 1e9
    GATHERS = ("k_gather_update_tc", "k_gather_update", "k_gather")
    PERSISTENT = ("k_sweep_fused", "k_sweep_wide")  # whole sweeps per launch

    def roofline_of(name):
        """HBM roofline of one kernel: algorithmic bytes per launch (the sampled fibers it gathers,
        B_eff x I_n x sizeof per SGD iteration) / its average CUDA-event duration."""
        if name in PERSISTENT:
            per_launch = prof_sweeps * fibers_per_step * (sum(cfg.dims) / N) * esz
        elif name in GATHERS:
            per_launch = gather_bytes
        else:
            return None
        t_k = kern[name]["avg_us"] * 1e-6
        ach = per_launch / t_k / 1e9
        # DRAM bytes (read + write) of this kernel from one ncu --set full capture (profiles/traffic.json,
        # written by tools/ncu_summary.py traffic): per launch, or per sweep for the fused kernel
        traffic = None
        tfile = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tfile):
            ent = json.load(open(tfile)).get(f"{cfg.name}/{args.sampler}/{name}")
            if ent:
                traffic = ent["bytes"] / ent.get("sweeps", 1) * (prof_sweeps if "sweeps" in ent else 1)
        return {"kernel": name, "bound": "hbm", "achieved": round(ach, 2), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": traffic,
                "frac_of_8TBs": round(ach / 8000.0, 4),  # also against the nominal ~8 TB/s
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "_fallback" not in peaks else "fallback",
                "algorithmic_bytes_per_launch": per_launch}

    roof = roofline_of(dominant) if dominant else None
    if roof is None and dominant is not None:
        # the dominant launch is the table/sampling kernel: a latency-bound serial chain (one cluster,
        # R sequential pivots), not a bandwidth kernel; report its share and the gather's roofline
        roof = {"kernel": dominant, "bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": None, "note": "dominant kernel is the per-step table rebuild + sampling chain "
                                         "(DESIGN.md 'Roofline'); see gather_roofline"}
    gather_roof = None
    for gname in GATHERS:
        if gname in kern:
            gather_roof = roofline_of(gname)
            break
    if roof is not None and dominant in PERSISTENT:
        roof["note"] = ("one launch runs every phase of every SGD iteration of the timed sweeps (sample -> gather -> "
                        "update -> table -> sample, serial by the method: R9); achieved = the sampled fibers' "
                        "bytes over the whole launch. The gather phase alone: phases.gather_roofline")
    # ---- e2e: host-buffer C-ABI call, H2D of all factors + D2H every step ----
    hflat = torch.empty(sum(a.numel() for a in Ad), dtype=Ad[0].dtype).pin_memory()  # one pinned block, views
    host, o = [], 0
    for a in Ad:
        v = hflat[o:o + a.numel()].view(a.shape)
        v.copy_(a.detach().cpu())
        host.append(v)
        o += a.numel()
    h2d = sum(a.numel() * esz for a in host)
    e2e_steps = max(2, min(args.steps, 20))
    for _ in range(max(2, min(args.warmup, 5))):  # untimed: first launches of the host-path kernels (lazy module loading)
        h.steps_host(0, N, host)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        h.steps_host(0, N, host)
    t1 = time.perf_counter()
    e2e_ms = (t1 - t0) * 1e3
    if ws > 1:
        import torch.distributed as dist

        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = fibers_per_step * e2e_steps * (1 if one_chain else ws) / (e2e_ms / 1e3)
    clocks = clk.summary()
    res = None
    if rank == 0:
        res = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": "strong" if one_chain else "weak", "vs_baseline": None,
            "dtype": "f64" if cfg.dtype == "f64" else "f32", "data": "synthetic (seeded; synth/ recipe)",
            "config": {"workload": workload_str(cfg, args.sampler),
                       "step": f"one cyclic sweep = {N} SGD iterations x B fibers",
                       "sampler": args.sampler,
                       "iterations_per_s": round(N * args.steps * (1 if one_chain else ws) / (ms / 1e3), 1),
                       "useful_GBps": round(useful_gbs, 2),
                       "layout": "native" if args.native_layout else "mode-major copies (CP_FLAG_MODE_MAJOR)",
                       "parallelism": (f"slab-sharded x{ws} (NCCL)" if sharded else
                                       f"one chain on {ws} whole-tensor replicas, batch split + "
                                       + ("M summed from peer memory in the update kernel" if p2p else "ncclAllReduce of M")
                                       if replica else (f"{ws} independent chains" if ws > 1 else "1 GPU")),
                       "l2": "inputs larger than L2 (tensor + mode-major copies >> 126 MB); fresh fibers per step",
                       "init_s": round(init_s, 3)},
            "roofline": roof,
            "gather_roofline": gather_roof,
            "kernels": {k: {"avg_us": round(v["avg_us"], 3), "share": round(v["share"], 4), "count": v["count"]}
                        for k, v in kern.items()},
            "kernel_timing": f"CUDA events around each launch on the library stream, {prof_sweeps} direct-launch sweeps",
            "path": h_path,
            "phases": None,
            "clocks": clocks,
            "e2e": {"value": round(e2e_val, 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": h2d,
                    "how": "cp_sgd_steps_host: pinned host factors -> device, one sweep, factors -> host, sync"},
            "gpu_launches": launches,
        }
    h.close()
    if res is not None and h_path == "persistent" and not args.no_phases:
        res["phases"] = phase_profile(args, cfg, Xd, Ad, stream, fibers_per_step / N, In_avg, esz, peaks)
    if res is not None and ws == 1 and args.other_samplers:
        res["other_samplers"] = other_samplers(args, cfg, Xd, Ad, stream, esz)
    return res


def other_samplers(args, cfg, Xd, Ad, stream, esz):
    """The same workload under the other sampling strategies (BASELINE configs[3]: "leverage-style and norm-style
    strategies"): fibers/s and us per cyclic sweep on the device clock (CUDA events, one launch per call), from the
    factors the headline run left.  Context next to the headline line, not a second headline."""
    import torch

    from paper_2103_04081_b200 import CPSGD

    out = {}
    K = max(5, min(args.steps, 100))
    for smp in [s for s in args.other_samplers.split(",") if s and s != args.sampler]:
        with torch.cuda.stream(stream):
            h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=smp, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta,
                      seed=cfg.seed, stream=stream, mode_major=not args.native_layout, fused=args.path == "auto",
                      tc=not args.no_tc)
        N = cfg.order
        fps = sum(h.batch_max(n) for n in range(N)) if smp.startswith("block") else N * cfg.batch
        h.sweep(max(3, args.warmup))
        h.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h.sweep(K)
        e1.record(stream)
        stream.synchronize()
        h.sync()
        ms = e0.elapsed_time(e1)
        out[smp] = {"value": round(fps * K / (ms / 1e3), 1), "unit": UNIT, "us_per_sweep": round(ms * 1e3 / K, 2),
                    "sweeps": K, "path": h.path,
                    "achieved_GBps": round(fps * K * (sum(cfg.dims) / N) * esz / (ms / 1e3) / 1e9, 2)}
        h.close()
    return out


def phase_profile(args, cfg, Xd, Ad, stream, fibers_per_iter, In_avg, esz, peaks, sweeps=3):
    """in-kernel phase timeline of the persistent wide kernel (CTA 0, clock64 at the phase boundaries; a
    second handle built with CPSGD_DEBUG_TIMERS on the same inputs, after the measured one): per SGD
    iteration, microseconds per phase, and the gather phase's HBM roofline (the sampled fibers' bytes /
    the time from the sampling barrier to the gather barrier, every CTA's gather included)"""
    import torch

    from paper_2103_04081_b200 import CPSGD

    os.environ["CPSGD_DEBUG_TIMERS"] = "1"
    try:
        with torch.cuda.stream(stream):
            h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=args.sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta,
                      seed=cfg.seed + 7, stream=stream, mode_major=not args.native_layout, fused=args.path == "auto",
                      tc=not args.no_tc)
    finally:
        del os.environ["CPSGD_DEBUG_TIMERS"]
    h.sweep(sweeps)
    h.sync()
    d = np.array(h.debug_timers()[512:512 + 256], dtype=np.int64).reshape(8, 32)
    h.close()
    its = [s for s in range(1, min(8, 3 * sweeps)) if d[s, 0] and d[s, 10] and d[s, 30] and d[s, 31]]
    if not its:
        return None
    ghz = float(np.mean([(d[s, 10] - d[s, 0]) / (d[s, 31] - d[s, 30]) for s in its]))
    seq = [("sample", 0, 1), ("barrier_S", 1, 2), ("gather", 2, 3), ("barrier_G", 3, 4), ("update", 4, 5),
           ("barrier_U", 5, 6), ("gram_pairs", 6, 7), ("inverse_scores_scan", 7, 9), ("barrier_Q", 9, 10)]
    out = {k: round(float(np.mean([(d[s, b] - d[s, a]) / ghz / 1e3 for s in its])), 2) for k, a, b in seq}
    out["iteration_us"] = round(float(np.mean([(d[s, 10] - d[s, 0]) / ghz / 1e3 for s in its])), 2)
    # BASELINE's "SGD steps/s per mode": iteration s of the launch updates mode s mod N (cyclic from 0)
    per = {}
    for s in its:
        per.setdefault(s % cfg.order, []).append((d[s, 10] - d[s, 0]) / ghz / 1e3)
    out["per_mode"] = {str(k): {"iteration_us": round(float(np.mean(v)), 2),
                                "steps_per_s": round(1e6 / float(np.mean(v)), 1)} for k, v in sorted(per.items())}
    t_g = float(np.mean([(d[s, 4] - d[s, 2]) / ghz for s in its])) * 1e-9
    ach = fibers_per_iter * In_avg * esz / t_g / 1e9
    out["gather_roofline"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                              "frac": round(ach / peaks["hbm_gbs"], 4),
                              "window": "sampling barrier -> gather barrier (every CTA's gather + the barrier)"}
    out["how"] = ("clock64 marks of CTA 0 at the phase boundaries of iterations 1..; CPSGD_DEBUG_TIMERS handle "
                  f"(SM clock {round(ghz * 1e3)} MHz)")
    return out


def cpu_baseline(cfg, args, budget_s=15.0, inputs=None):
    """the oracle as it stands (single thread, fp64 arithmetic) on a bounded sample of the same workload:
    whole SGD iterations (one mode update of B fibers each, cyclic modes) until ~budget_s of CPU time"""
    import oracle

    X, A0 = inputs if inputs is not None else host_inputs(cfg)
    st = oracle.STRATEGIES[args.sampler]
    rule = {"adaptive": oracle.STEP_ADAPTIVE, "als": oracle.STEP_ALS}.get(cfg.rule, oracle.STEP_FIXED)
    iters, t_used = 0, 0.0
    fs, S = A0, None
    while t_used < budget_s and iters < 3 * 200:
        t0 = time.perf_counter()
        fs, S, _ = oracle.run(X, fs, st, rule, cfg.batch, 1, alpha=cfg.alpha, eta=cfg.eta, seed=cfg.seed, r0=iters,
                              S=S, first_mode=iters % cfg.order)
        t_used += time.perf_counter() - t0
        iters += 1
    fib = iters * cfg.batch
    return {"value": round(fib / t_used, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{iters} oracle SGD iterations (cyclic modes from 0, B = {cfg.batch} fibers each) of "
                      f"{workload_str(cfg, args.sampler)}; fp64 single-threaded C (-O2), tensor host-resident "
                      f"({'fp32, read in place' if X.dtype == np.float32 else 'fp64'}); per-iteration table rebuild "
                      f"by Householder QR included", "seconds": round(t_used, 2), "host": host_info()}


def run_reference(args, cfg):
    """the reference arm: the CPU oracle (there is no reference implementation: the paper is the
    reference) on the same workload, one SGD iteration of B fibers per step, rank 0 only"""
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    import oracle

    X, A0 = host_inputs(cfg)
    st = oracle.STRATEGIES[args.sampler]
    rule = {"adaptive": oracle.STEP_ADAPTIVE, "als": oracle.STEP_ALS}.get(cfg.rule, oracle.STEP_FIXED)
    fs, S = A0, None
    r = 0
    for _ in range(args.warmup):
        fs, S, _ = oracle.run(X, fs, st, rule, cfg.batch, 1, alpha=cfg.alpha, eta=cfg.eta, seed=cfg.seed, r0=r, S=S,
                              first_mode=r % cfg.order)
        r += 1
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fs, S, _ = oracle.run(X, fs, st, rule, cfg.batch, 1, alpha=cfg.alpha, eta=cfg.eta, seed=cfg.seed, r0=r, S=S,
                              first_mode=r % cfg.order)
        r += 1
    dt = time.perf_counter() - t0
    fib = args.steps * cfg.batch
    val = fib / dt
    return {"impl": "reference", "metric": METRIC, "value": round(val, 1), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * dt / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; synth/ recipe)",
            "config": {"workload": workload_str(cfg, args.sampler),
                       "step": f"one SGD iteration = B = {cfg.batch} fibers (modes cyclic)"},
            "cpu_baseline": {"value": round(val, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} SGD iterations of {cfg.name} (fp64 oracle, single thread)",
                             "host": host_info()},
            "e2e": {"value": round(val, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4", choices=list(synth.CONFIGS))
    ap.add_argument("--sampler", default="leverage",
                    choices=["uniform", "leverage", "euclidean", "block_leverage", "block_euclidean"])
    ap.add_argument("--native-layout", action="store_true", help="no mode-major copies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--other-samplers", default="euclidean,uniform",
                    help="comma list of strategies also timed on the same workload (N = 1; '' to skip)")
    ap.add_argument("--no-phases", action="store_true", help="skip the in-kernel phase timeline of the persistent kernel")
    ap.add_argument("--path", default="auto", choices=["auto", "wide"],
                    help="auto: persistent single-cluster kernel when the problem fits one cluster; wide: the "
                         "gather (tcgen05) + table/sampling kernel pair")
    ap.add_argument("--no-tc", action="store_true", help="FFMA gather mainloop instead of tcgen05")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1 replicas: M by ncclAllReduce, or over peer memory summed inside the update kernel "
                         "(CP_FLAG_P2P, IPC-mapped symmetric buffers)")
    ap.add_argument("--independent", action="store_true",
                    help="N > 1: one unrelated chain per GPU (weak scaling) instead of one chain on N replicas")
    ap.add_argument("--chains", type=int, default=1,
                    help="K > 1: K independent chains in one multi-chain launch (fused workloads; SURVEY 8f.2)")
    ap.add_argument("--chain-cluster", type=int, default=16, choices=[8, 16],
                    help="--chains: CTAs per chain (8: two chains per GPC)")
    ap.add_argument("--slab-of", type=int, default=0,
                    help="P > 1: time rank 0's share of a P-way slab-sharded run on one GPU (exchanges excluded)")
    ap.add_argument("--rule", default="config", choices=["config", "fixed", "adaptive", "als"],
                    help="update rule (config: the workload's; als: the sampled least-squares step, SURVEY 8f.3)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = synth.CONFIGS[args.workload]
    if args.rule != "config":
        import dataclasses

        cfg = dataclasses.replace(cfg, rule=args.rule)
    if args.impl == "reference":
        res = run_reference(args, cfg)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    import __graft_entry__

    ws, rank, _ = dist_env()
    __graft_entry__.build()  # idempotent (mtime check, atomic replace)
    if args.chains > 1:
        print(json.dumps(run_chains(args, cfg)), flush=True)
        return
    if args.slab_of > 1:
        print(json.dumps(run_slab(args, cfg)), flush=True)
        return
    if ws > 1:
        import torch.distributed  # noqa: F401
    res = run_ours(args, cfg)
    if rank == 0:
        if not args.no_cpu_baseline and ws == 1:
            res["cpu_baseline"] = cpu_baseline(cfg, args)
        print(json.dumps(res), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
