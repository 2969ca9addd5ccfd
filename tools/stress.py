"""Determinism / race stress on cuda:0: every path runs the same long trajectory twice and must agree
bit for bit (a race in a cluster kernel shows up as a mismatch or a launch failure).

C2 (fused 16-CTA, fused 8-CTA, wide), C3 (fused), C4 (wide, tcgen05): 60 sweeps each, twice; then
14 chains of C2 in one launch (8-CTA clusters), 50 sweeps, against a second multi-chain run.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402

dev = torch.device("cuda:0")
SWEEPS = int(os.environ.get("STRESS_SWEEPS", "60"))


def problem(name):
    cfg = synth.CONFIGS[name]
    if cfg.numel <= 200_000_000:
        X = synth.tensor(cfg)
        A0 = synth.init_factors(cfg, X)
        Xd = torch.from_numpy(X).to(dev)
        A0d = [torch.from_numpy(a).to(dev) for a in A0]
    else:
        Xd, _, xn = synth.tensor_torch(cfg, device=dev)
        A0d = synth.init_factors_torch(cfg, xn, device=dev)
    return cfg, Xd, A0d


def run(cfg, Xd, A0d, sampler, **kw):
    Ad = [a.clone() for a in A0d]
    h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta, seed=3, **kw)
    h.sweep(SWEEPS)
    h.sync()
    h.close()
    return [a.cpu() for a in Ad]


bad = 0
t0 = time.time()
for name, variants in [("C2", [dict(), dict(fused_cluster=8), dict(fused=False)]), ("C3", [dict()]),
                       ("C4", [dict()])]:
    cfg, Xd, A0d = problem(name)
    for sampler in (["leverage", "euclidean", "block_leverage", "uniform"] if name != "C4" else ["leverage", "euclidean", "block_euclidean"]):
        for kw in variants:
            a = run(cfg, Xd, A0d, sampler, **kw)
            b = run(cfg, Xd, A0d, sampler, **kw)
            same = all(torch.equal(x, y) for x, y in zip(a, b))
            bad += not same
            print(f"{name} {sampler:15s} {str(kw):22s} {'ok' if same else 'MISMATCH'}", flush=True)
    del Xd, A0d
    torch.cuda.empty_cache()

cfg, Xd, A0d = problem("C2")
outs = []
for rep in range(2):
    hs, As = [], []
    for c in range(14):
        Ad = [a.clone() for a in A0d]
        hs.append(CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler="leverage", rule=cfg.rule, eta=cfg.eta, seed=c,
                        fused_cluster=8))
        As.append(Ad)
    CPSGD.sweep_multi(hs, 50)
    for h in hs:
        h.sync()
        h.close()
    outs.append([[a.cpu() for a in Ad] for Ad in As])
same = all(torch.equal(x, y) for ca, cb in zip(*outs) for x, y in zip(ca, cb))
bad += not same
print(f"C2 14 chains x 50 sweeps {'ok' if same else 'MISMATCH'}")
print(f"stress: {bad} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
