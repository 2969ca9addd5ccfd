"""Run a few sweeps of a BASELINE config on cuda:0 (profiling driver for ncu / sanitizers)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
ap.add_argument("--sampler", default="leverage")
ap.add_argument("--sweeps", type=int, default=5)
ap.add_argument("--direct", action="store_true", help="no CUDA graph")
ap.add_argument("--wide", type=int, default=1, help="0: legacy split path (gather partials + update/table)")
ap.add_argument("--fused", type=int, default=1)
a = ap.parse_args()
cfg = synth.CONFIGS[a.workload]
dev = torch.device("cuda:0")
if cfg.numel <= 200_000_000:
    X = synth.tensor(cfg)
    A0 = synth.init_factors(cfg, X)
    Xd = torch.from_numpy(X).to(dev)
    Ad = [torch.from_numpy(x).to(dev) for x in A0]
else:
    Xd, _, xn = synth.tensor_torch(cfg, device=dev)
    Ad = synth.init_factors_torch(cfg, xn, device=dev)
h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=a.sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta, seed=0,
          graphs=not a.direct, wide=bool(a.wide), fused=bool(a.fused))
h.sweep(2)
h.sync()
t = time.perf_counter()
h.sweep(a.sweeps)
h.sync()
print(f"{a.workload} {a.sampler}: {(time.perf_counter() - t) / a.sweeps * 1e6:.1f} us/sweep")
if a.direct:
    h.profile(True)
    h.sweep(a.sweeps)
    prof = h.profile_read()
    h.profile(False)
    print("  per launch (CUDA events): " + ", ".join(f"{k} {v[0] / v[1] * 1e3:.1f} us x{v[1]}" for k, v in prof.items()))
h.close()
if os.environ.get("CPSGD_DEBUG_TIMERS") and os.environ.get("FUSED_TIMERS"):
    h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=a.sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta, seed=0)
    h.sweep(1)
    t = h.debug_timers()
    names = ["gather", "sync1", "reduce+update", "gram-part", "sync2", "gram-sum+sweep", "scores", "scan", "sync3",
             "cdf", "sync4", "sample"]
    print(" | ".join(f"{names[i]}:{t[i + 1] - t[i]}" for i in range(12)), "| total", t[12] - t[0])
    print("gram-sum", t[13] - t[5], "sweep", t[6] - t[13], "| gather: contract", t[14] - t[0], "Gamma part", t[15] - t[14],
          "Aold", t[1] - t[15])
    print("  sample: draws", t[24] - t[23], "weights/offsets", t[25] - t[24], "cp.async issue", t[26] - t[25], "SKR", t[27] - t[26])
    print("  contract: ld0", t[17] - t[16], "fma0", t[18] - t[17], "ld1", t[19] - t[18], "fma1", t[20] - t[19], "store", t[14] - t[20])
elif os.environ.get("CPSGD_DEBUG_TIMERS"):
    h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=a.sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta, seed=0,
              graphs=False, wide=bool(a.wide), fused=bool(a.fused))
    h.sweep(3)
    t = h.debug_timers()
    if t[36]:
        print("k_gather_update_tc cycles: prologue", t[33] - t[32], "mainloop", t[34] - t[33], "tmem->smem", t[35] - t[34],
              "finish", t[36] - t[35])
        import numpy as np
        g0 = np.array(t[1024:3072:2]); g1 = np.array(t[1025:3072:2]); m = g0 > 0
        g0, g1 = g0[m], g1[m]
        base = g0.min()
        print(f"  CTAs {m.sum()}: start spread {(g0.max() - base) / 1e3:.1f} us, end min {(g1.min() - base) / 1e3:.1f} "
              f"max {(g1.max() - base) / 1e3:.1f} us, duration median {np.median(g1 - g0) / 1e3:.1f} us; "
              f"distinct SMs {len(set(t[3072:3072 + m.sum()]))}")
        print("  stage 8: load issue->data", t[18] - t[23], "wait xh/xl", t[19] - t[18], "split", t[20] - t[19],
              "split->mma start", t[21] - t[20], "mma issue", t[22] - t[21], "| mma thread: wait sdone", t[25] - t[24],
              "wait A image", t[21] - t[25], "| split: wait xfull", t[18] - t[26], "stage 8->9", t[27] - t[26],
              "stage 8->12 /4", (t[28] - t[26]) / 4)
    if t[107]:
        nm = ["cdf stage", "draw", "skr", "zw/img", "gamma", "cluster+fence", "last"]
        print("k_sample_wide (CTA 0) cycles: " + " | ".join(f"{nm[i]} {t[101 + i] - t[100 + i]}" for i in range(7)))
        print("  gamma: own blocks", t[108] - t[104], "barrier", t[109] - t[108], "group sum", t[105] - t[109])
        import numpy as np
        g0 = np.array(t[2048:3008:2]); g1 = np.array(t[2049:3008:2]); m = g0 > 0
        g0, g1 = g0[m], g1[m]
        base = g0.min()
        print(f"  k_sample_wide CTAs {m.sum()}: start spread {(g0.max() - base) / 1e3:.1f} us, end min "
              f"{(g1.min() - base) / 1e3:.1f} max {(g1.max() - base) / 1e3:.1f} us, median dur {np.median(g1 - g0) / 1e3:.1f} us")
    if t[317]:
        print("k_update_wide (ns, globaltimer): CTA0 body", t[311] - t[310], "| last CTA: starts", t[312] - t[310],
              "Gram gather", t[313] - t[312], "sweep", t[314] - t[313], "W write", t[315] - t[314])
        print("  CTA0: W wait ends", t[316] - t[310], "scores+scan", t[317] - t[316])
    if not a.wide:
        names = ["start", "stageB", "gram-synced", "sweep-start", "sweep-done", "scores-done", "cdf-synced", "sampled"]
        print(" ".join(f"{names[i]}:{t[i] - t[0]}" for i in range(8)))
