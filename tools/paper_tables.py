"""the paper's Table 1 / Table 2 experiment, qualitatively (orderings only; the
paper's numbers are seed-, generator- and hardware-specific and are not reproduced).

I x I x 15 tensors, R = 25, batch |F_n| = 18, U[0,1] initial factors exactly as the paper states (
--init scaled: norm-matched to ||X||, reading R13), adaptive step (Alg. 7,
b = eps = 0), spread = 15, magnitude = 24, 5 % noise, generator:
synth.spread_magnitude (SPEC.md's stand-in for the cited rule).  For each sampler and seed the
library runs on cuda:0 (fused path); after every iteration (one mode update) the relative errors
  e_X  = ||X - [[A]]|| / ||X||          (cp_fit)
  e_0  = ||X0 - [[A]]|| / ||X0||        (against the clean tensor; host-side, from the factors)
are recorded.  Reported per sampler (median over seeds):
  Table 1: iterations until |e_X(r) - e_X(r-1)| < tol = 1e-4 (cap 3000);
  Table 2: e_0 after `it` iterations (I = 100: 55).
Prints one JSON line per I and writes it to profiles/ when --out is given.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--I", type=int, default=100)
ap.add_argument("--it", type=int, default=55)
ap.add_argument("--seeds", type=int, default=10)
ap.add_argument("--eta", type=float, default=0.05)
ap.add_argument("--cap", type=int, default=3000)
ap.add_argument("--tol", type=float, default=1e-4)
ap.add_argument("--out", default="")
ap.add_argument("--init", default="raw", choices=["raw", "scaled"])
ap.add_argument("--checkpoints", default="55,80,200,500,1000,1500,3000")
a = ap.parse_args()
dev = torch.device("cuda:0")
R, J, B = 25, 15, 18
samplers = ["uniform", "euclidean", "leverage", "block_euclidean", "block_leverage"]
cps = sorted({int(c) for c in a.checkpoints.split(",") if int(c) <= a.cap} | {a.it})
res = {s: {"iters": [], "err0": {c: [] for c in cps}} for s in samplers}
for seed in range(a.seeds):
    X, X0, _ = synth.spread_magnitude(a.I, J, R, 15, 24.0, 0.05, seed=seed)  # I x I x J
    dims = (a.I, a.I, J)
    rng = np.random.default_rng([seed, 5])
    A0 = [rng.random((d, R)) for d in dims]
    if a.init == "scaled":  # U[0,1] factors norm-matched to ||X|| (reading R13)
        H = np.ones((R, R))
        for A in A0:
            H = H * (A.T @ A)
        sc = (np.linalg.norm(X) / np.sqrt(H.sum())) ** (1.0 / 3.0)
        A0 = [A * sc for A in A0]
    n0 = np.linalg.norm(X0)
    for s in samplers:
        Xd = torch.from_numpy(X).to(dev)
        Ad = [torch.from_numpy(A.copy()).to(dev) for A in A0]
        h = CPSGD(Xd, dims, Ad, B, sampler=s, rule="adaptive", eta=a.eta, b=0.0, eps=0.0, seed=seed)
        prev, iters = None, None
        for r in range(1, a.cap + 1):
            h.step((r - 1) % 3)
            eX = 1.0 - h.fit()
            if r in res[s]["err0"]:
                F = [A.cpu().numpy() for A in Ad]
                res[s]["err0"][r].append(float(np.linalg.norm(X0 - synth.cp_tensor(F)) / n0))
            if iters is None and prev is not None and abs(eX - prev) < a.tol:
                iters = r
            prev = eX
        res[s]["iters"].append(iters if iters is not None else a.cap)
        h.close()
summary = {"I": a.I, "J": J, "R": R, "B": B, "eta": a.eta, "tol": a.tol, "init": a.init, "seeds": a.seeds,
           "iteration": "one mode update of |F_n| = B fibers (cyclic modes)",
           "error": "||X0 - [[A]]|| / ||X0|| against the clean tensor",
           "median_iters_to_tol": {s: float(np.median(res[s]["iters"])) for s in samplers},
           "median_err_clean": {str(c): {s: float(np.median(res[s]["err0"][c])) for s in samplers} for c in cps}}
last = summary["median_err_clean"][str(cps[-1])]
summary["orderings_at_cap"] = {"euclidean<uniform": last["euclidean"] < last["uniform"],
                               "leverage<uniform": last["leverage"] < last["uniform"],
                               "max(E,L)<min(BE,BL)": max(last["euclidean"], last["leverage"]) <
                               min(last["block_euclidean"], last["block_leverage"])}
print(json.dumps(summary))
if a.out:
    with open(a.out, "w") as f:
        f.write(json.dumps(summary, indent=1) + "\n")
