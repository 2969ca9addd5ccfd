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


def row_rel_err(a, b, floor_frac=1e-2):
    """max over rows of ||a_i - b_i|| / (||b_i|| + floor), floor = floor_frac x the mean row norm of b:
    a per-row bound next to the Frobenius one (a large error in one row cannot hide in the norm)"""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    rn = np.linalg.norm(b, axis=1)
    floor = floor_frac * max(float(rn.mean()), 1e-300)
    return float(np.max(np.linalg.norm(a - b, axis=1) / (rn + floor)))


def q_of_cdf(cdf):
    c = np.asarray(cdf, np.uint64)
    return np.diff(np.concatenate([np.zeros(1, np.uint64), c])).astype(np.uint64)


def trace_check(X, dims, A0, recs, strategy, B, seed, rule, cfg, q_init, alphas=None, tol=None, b=0.0, S0=None,
                grad=None):
    """Teacher-forced check of a cp_sgd_trace record list (tests/test_gpu_persistent.py):
    for every iteration s, from the traced state before it (factors, accumulators and integer tables
    as the GPU left them):
      (1) the batch: idx and w bit-exact with oracle.sample on the GPU's integer tables;
      (2) the update: the oracle's gradient on that batch and its fixed / adaptive step equal the
          traced A^(n) (and S^(n)) within tol.  b = 0 makes an AdaGrad step eta sign(G) where S was 0:
          such entries whose oracle |G| lies inside the band 10 tol (||A Gamma|| + ||M||) / sqrt(I_n R)
          (an fp32 G error that large could flip the sign) are masked, and must be < 5 % of the entries;
      (3) the rebuilt table: q = diff(traced CDF) equals the oracle's table of the traced factor except
          entries within 1e-3 of a rounding boundary (|dq| <= 1 there).
    Returns the number of masked entries."""
    st = oracle.STRATEGIES[strategy]
    tol = TOL["f32"] if tol is None else tol
    A = [np.asarray(a, np.float64).copy() for a in A0]
    Sacc = [np.zeros_like(a) for a in A] if S0 is None else [np.asarray(s, np.float64).copy() for s in S0]
    q = [np.asarray(x, np.uint64) for x in q_init]
    masked = 0
    for s, rec in enumerate(recs):
        n, r = rec["n"], rec["r"]
        tq = [(q[k], int(q[k].sum())) for k in range(len(dims))]
        idx_o, w_o, pj = oracle.sample(dims, n, st, B, tq, seed, r)
        assert np.array_equal(rec["idx"], idx_o), f"iteration {s}: indices differ"
        assert np.array_equal(rec["w"], w_o), f"iteration {s}: weights differ"
        if grad is None:
            G_o, Gam_o, M_o = oracle.gradient(X, dims, A, n, st, B, idx_o, pj)
        else:  # tensors too large for the oracle's own TensorSamp: fibers read from the seeded input
            G_o, Gam_o, M_o = grad(A, n, idx_o, pj)
        scale = np.linalg.norm(A[n] @ Gam_o) + np.linalg.norm(M_o)
        A_g = np.asarray(rec["A"], np.float64)
        if rule == "fixed":
            al = cfg.alpha if alphas is None else float(alphas[s])
            A_o = oracle.update_fixed(A[n], G_o, al)
            assert rel_err(A_g, A_o, np.linalg.norm(A_o)) <= tol, f"iteration {s}: A"
            assert row_rel_err(A_g, A_o) <= 10 * tol, f"iteration {s}: A rows"
        else:
            A_o, S_o = oracle.update_adaptive(A[n], Sacc[n], G_o, cfg.eta, b=b)
            S_g = np.asarray(rec["S"], np.float64)
            assert rel_err(S_g, S_o, np.linalg.norm(S_o)) <= 2 * tol, f"iteration {s}: S"
            # sign-sensitive entries: never updated before (S = 0: the step is eta sign(G)) and |G| inside
            # the band an fp32 G error could cross
            band = (Sacc[n] == 0.0) & (np.abs(G_o) <= 10 * tol * scale / np.sqrt(G_o.size))
            masked += int(band.sum())
            assert band.mean() < 0.05, f"iteration {s}: {band.mean():.3%} of the entries masked"
            d = np.where(band, 0.0, A_g - A_o)
            assert np.linalg.norm(d) <= tol * np.linalg.norm(A_o), f"iteration {s}: A (masked)"
            assert row_rel_err(np.where(band, A_o, A_g), A_o) <= 10 * tol, f"iteration {s}: A rows (masked)"
            Sacc[n] = S_g
        qg = q_of_cdf(rec["cdf"])
        po, qo, _ = oracle.build_table(st, A_g)
        diff = qg != qo
        assert np.all(~diff | near_boundary(po, 1e-3)), f"iteration {s}: table"
        assert np.all(np.abs(qg.astype(np.int64) - qo.astype(np.int64)) <= 1)
        A[n] = A_g
        q[n] = qg
    return masked
