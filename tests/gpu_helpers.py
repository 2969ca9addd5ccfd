"""Shared setup for the GPU parity tests: seeded inputs (synth), oracle references, tolerances.

Every oracle input comes from synth (the seeded generators) -- never from the CUDA path.
"""
import numpy as np

import oracle
import synth

S = ["uniform", "leverage", "euclidean", "block_leverage", "block_euclidean"]

# tolerances: fp64 1e-10, fp32 1e-4 relative, per BASELINE north_star
TOL = {"f64": 1e-10, "f32": 1e-4}


def torch_dev():
    import torch

    return torch.device("cuda:0")


def make_problem(cfg, seed=None):
    X = synth.tensor(cfg, seed)
    A0 = synth.init_factors(cfg, X, seed)
    return X, A0


def to_dev(X, A0):
    import torch

    dev = torch_dev()
    return torch.from_numpy(X).to(dev), [torch.from_numpy(np.ascontiguousarray(A)).to(dev) for A in A0]


def handle(cfg, Xd, Ad, sampler, **kw):
    from paper_2103_04081_b200 import CPSGD

    args = dict(sampler=sampler, rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta, seed=kw.pop("seed", 0))
    args.update(kw)
    return CPSGD(Xd, cfg.dims, Ad, cfg.batch, **args)


def oracle_tables(strategy, factors):
    st = oracle.STRATEGIES[strategy]
    out = []
    for A in factors:
        p, q, T = oracle.build_table(st, np.asarray(A, dtype=np.float64))
        out.append((p, q, T))
    return out


def rel_err(a, b, scale):
    return float(np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / max(scale, 1e-300))


def oracle_step(X, dims, factors, n, strategy, B, seed, it, window=None):
    """one oracle iteration from the given (synth) factors; returns idx, w, G, Gamma, M."""
    tabs = oracle_tables(strategy, factors)
    tq = [(t[1], t[2]) for t in tabs]
    st = oracle.STRATEGIES[strategy]
    idx, w, pj = oracle.sample(dims, n, st, B, tq, seed, it, window)
    G, Gam, M = oracle.gradient(X, dims, [np.asarray(A, np.float64) for A in factors], n, st, B, idx, pj)
    return idx, w, G, Gam, M, tabs


def near_boundary(p, tol_abs):
    """entries whose fixed-point value p 2^32 lies within tol_abs of a rounding boundary (x.5)"""
    s = np.asarray(p, np.float64) * 2.0 ** 32
    return np.abs(s - np.floor(s) - 0.5) <= tol_abs


def gather_fibers_torch(Xd, dims, n, idx):
    """X_(n)(:, F) as a (B, I_n) fp64 array read from the seeded input tensor on the device (input
    data from synth, first-index-fastest layout -- not an output of the CUDA path)."""
    import torch

    strides = np.cumprod([1] + list(dims[:-1])).astype(np.int64)
    base = np.zeros(idx.shape[0], np.int64)
    pos = 0
    for k in range(len(dims)):
        if k == n:
            continue
        base += idx[:, pos].astype(np.int64) * strides[k]
        pos += 1
    off = (torch.from_numpy(base).to(Xd.device)[:, None]
           + torch.arange(dims[n], device=Xd.device, dtype=torch.int64)[None, :] * int(strides[n]))
    return Xd[off].double().cpu().numpy()


def oracle_gradient_from_fibers(XF, dims, factors, n, strategy, B, idx, pj):
    """eq:gradient1/2 for row-wise strategies from pre-gathered fibers XF (B, I_n):
    the oracle's SKR rows (oracle.skr), D = diag(1/p_j) and the 1/(B J_n) scale of oracle.gradient,
    for problems whose full tensor does not fit the oracle.  Pinned against oracle.gradient in
    tests/test_oracle_pins.py::test_gradient_from_fibers_matches_oracle."""
    assert strategy in ("uniform", "leverage", "euclidean")
    fs = [np.asarray(A, np.float64) for A in factors]
    Z = oracle.skr(fs, n, idx)
    Jn = float(np.prod([d for k, d in enumerate(dims) if k != n]))
    scale = 1.0 / (float(B) * Jn)
    d = 1.0 / np.asarray(pj, np.float64)
    C1 = Z.T @ (d[:, None] * Z)
    C2 = np.asarray(XF, np.float64).T @ (d[:, None] * Z)
    Gam = scale * C1
    M = scale * C2
    G = scale * (fs[n] @ C1 - C2)
    return G, Gam, M
