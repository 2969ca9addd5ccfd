"""Per-CTA phase durations of the persistent wide kernel (CPSGD_DEBUG_TIMERS; clock64 differences inside
each CTA, so no cross-SM clock alignment is needed): for every phase, CTA 0 / median / max over CTAs and
the CTA with the max, averaged over iterations 1..7 -- the max column is the phase's share of the critical
path (every phase ends at a grid-wide synchronisation).  python tools/pw_cta.py [C4|C2]"""
import os
import sys

os.environ["CPSGD_DEBUG_TIMERS"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = synth.CONFIGS[name]
dev = torch.device("cuda:0")
if cfg.numel > 2e8:
    Xd, _, xn = synth.tensor_torch(cfg, device=dev)
    Ad = synth.init_factors_torch(cfg, xn, device=dev)
else:
    X = synth.tensor(cfg)
    Xd = torch.from_numpy(X).to(dev)
    Ad = [torch.from_numpy(a).to(dev) for a in synth.init_factors(cfg, X)]
h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler="leverage", rule=cfg.rule, eta=cfg.eta, seed=1, fused=False)
assert h.path == "persistent"
h.sweep(3)
h.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(h.stream)
h.sweep(20)
e1.record(h.stream)
h.sync()
print("us/sweep", round(e0.elapsed_time(e1) * 1e3 / 20, 2))
h.sweep(3)
h.sync()
d = np.array(h.debug_timers(), dtype=np.int64)
ghz_t = d[512:512 + 256].reshape(8, 32)
ghz = float(np.mean([(ghz_t[s, 10] - ghz_t[s, 0]) / (ghz_t[s, 31] - ghz_t[s, 30]) for s in range(1, 8)]))
m = d[4096:4096 + 8 * 160 * 32].reshape(8, 160, 32)
G = int((m[1, :, 0] != 0).sum())
m = m[:, :G, :]
seq = [("S", 0, 1), ("wait S", 1, 2), ("G", 2, 3), ("wait G", 3, 4), ("U", 4, 5), ("wait U", 5, 6), ("P", 6, 7),
       ("wait P", 7, 18), ("Gram load", 18, 19), ("inverse", 19, 20), ("-> Q", 20, 8), ("Q", 8, 9), ("wait Q", 9, 10)]
print(f"{G} CTAs, SM clock {ghz * 1e3:.0f} MHz; us, mean over iterations 1..7")
print(f"  {'phase':10s} {'CTA0':>7s} {'median':>7s} {'max':>7s}  argmax")
tot_max = 0.0
for nm, a, b in seq:
    v = m[1:8, :, b] - m[1:8, :, a]
    ok = (m[1:8, :, a] != 0) & (m[1:8, :, b] != 0)
    v = np.where(ok, v, np.nan) / ghz / 1e3
    mean = np.nanmean(v, axis=0)  # per CTA
    if np.all(np.isnan(mean)):
        continue
    c0 = mean[0]
    mx = np.nanmax(mean)
    tot_max += mx if not nm.startswith("wait") else 0.0
    print(f"  {nm:10s} {c0:7.2f} {np.nanmedian(mean):7.2f} {mx:7.2f}  {int(np.nanargmax(mean))}")
print(f"  sum of the non-wait maxima: {tot_max:.2f} us (iteration total at CTA 0: "
      f"{float((ghz_t[1:8, 31] - ghz_t[1:8, 30]).mean()) / 1e3:.2f} us)")
