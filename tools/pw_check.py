"""Quick GPU check of the persistent wide sweep kernel (k_sweep_wide) against the kernel chain and the
oracle on a C4-shaped small problem: one step per mode from the same seeded state, then a few sweeps
(trace of the consumed batches compared with oracle.sample on the traced tables)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402


def main():
    dims = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "300,260,200").split(","))
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
    strategy = sys.argv[4] if len(sys.argv) > 4 else "leverage"
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule="adaptive", row_sigma=1.0, noise=1e-2, seed=3, eta=0.03)
    X = synth.tensor(cfg)
    A0 = synth.init_factors(cfg, X)
    dev = torch.device("cuda:0")
    Xd = torch.from_numpy(X).to(dev)
    res = {}
    for persist in (True, False):
        Ad = [torch.from_numpy(a.copy()).to(dev) for a in A0]
        h = CPSGD(Xd, dims, Ad, B, sampler=strategy, rule="adaptive", eta=0.03, seed=7, fused=False, persist=persist)
        print("path", h.path, flush=True)
        if persist:
            h.trace_start(12)
        h.sweep(4)
        h.sync()
        res[persist] = [a.cpu().numpy() for a in Ad]
        if persist:
            tr = h.trace_read()
        t0 = time.time()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h.stream)
        h.sweep(20)
        e1.record(h.stream)
        h.sync()
        print("persist" if persist else "chain", "us/sweep", e0.elapsed_time(e1) * 1e3 / 20, flush=True)
        h.close()
    for k in range(3):
        a, b = res[True][k].astype(np.float64), res[False][k].astype(np.float64)
        print("mode", k, "persist vs chain rel", np.linalg.norm(a - b) / np.linalg.norm(b))
    # trace: batches equal oracle.sample from the traced tables
    A = [a.astype(np.float64) for a in A0]
    st = oracle.STRATEGIES[strategy]
    tabs = [oracle.build_table(st, a) for a in A]
    q = [t[1] for t in tabs]
    T = [t[2] for t in tabs]
    bad = 0
    for s, rec in enumerate(tr):
        n = rec["n"]
        idx_o, w_o, _ = oracle.sample(dims, n, st, B, [(q[k], T[k]) for k in range(3)], 7, rec["r"])
        ok = np.array_equal(idx_o, rec["idx"]) and np.array_equal(w_o, rec["w"])
        cdf = rec["cdf"]
        qg = np.diff(np.concatenate([[0], cdf.astype(np.uint64)])).astype(np.uint64)
        _, qo, To = oracle.build_table(st, rec["A"].astype(np.float64))
        flips = int((qg != qo).sum())
        print("step", s, "n", n, "r", rec["r"], "batch bit-exact", ok, "table flips vs oracle(traced A)", flips)
        bad += (not ok)
        q[n] = qg
        T[n] = int(cdf[-1])
    print("BAD" if bad else "OK")


if __name__ == "__main__":
    main()
