"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs C1-C5).

This module is the ONE piece shared by the oracle side and the CUDA side: it only draws
random numbers and assembles the dense tensor X = [[A_true]] + noise (the CP model,
PAPER.md:27-33) plus the initial factors.  It holds none of the method's arithmetic
(no sampling, tables, gradients or updates).

Recipes (readings R13, R15, R22):
  factors  : entries N(0,1); each row scaled by exp(N(0, row_sigma)); optional unit-norm
             columns (C2); optional column congruence c via A = G L^T, L = chol((1-c)I + c 11^T)
             applied before the row scaling (C3).
  tensor   : X0 = [[A_true]] stored first-index-fastest;
             X = X0 + rho * (||X0||_F / ||E||_F) * E, E iid N(0,1)  (exact noise ratio).
  init     : U[0,1] entries, then every factor scaled by
             (||X||_F / ||[[A0]]||_F)^(1/N) (reading R13).

Two backends with identical recipes (different random streams): ``numpy`` (host, small and
medium tensors; used by every parity test) and ``torch`` on a CUDA device (large tensors,
generated in slabs along the last mode).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    dims: tuple
    rank: int
    dtype: str            # "f32" | "f64"
    batch: int
    rule: str             # "fixed" | "adaptive"
    row_sigma: float = 1.0
    unit_columns: bool = False
    congruence: float = 0.0
    noise: float = 1e-2
    alpha: float = 0.01   # fixed rule
    eta: float = 0.05     # adaptive rule
    sampler: str = "leverage"
    seed: int = 0

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def itemsize(self) -> int:
        return 8 if self.dtype == "f64" else 4

    @property
    def numel(self) -> int:
        return int(np.prod(self.dims))


# BASELINE.json configs, index-aligned (configs[0] .. configs[4]).
CONFIGS = {
    "C1": Config("C1", (60, 60, 60), 5, "f64", 64, "fixed", row_sigma=1.0, noise=1e-2, alpha=0.002),
    "C2": Config("C2", (400, 400, 400), 20, "f32", 512, "adaptive", row_sigma=1.5, unit_columns=True, noise=1e-2,
                 eta=0.03),
    "C3": Config("C3", (100, 100, 100, 100), 10, "f32", 1024, "adaptive", row_sigma=1.0, congruence=0.9,
                 noise=1e-3, eta=0.03),
    "C4": Config("C4", (2000, 2000, 2000), 50, "f32", 4096, "adaptive", row_sigma=1.0, noise=1e-2, eta=0.03),
    "C5": Config("C5", (4000, 4000, 4000), 32, "f32", 8192, "adaptive", row_sigma=1.0, noise=1e-2, eta=0.03),
}


def small(dims, rank, dtype="f64", batch=16, **kw) -> Config:
    """A small ad-hoc config for parity tests."""
    return Config("small", tuple(int(d) for d in dims), int(rank), dtype, int(batch), kw.pop("rule", "fixed"), **kw)


def true_factors(cfg: Config, seed: Optional[int] = None) -> List[np.ndarray]:
    rng = np.random.default_rng([cfg.seed if seed is None else seed, 1])
    out = []
    for I in cfg.dims:
        G = rng.standard_normal((I, cfg.rank))
        if cfg.congruence > 0.0:
            c = cfg.congruence
            L = np.linalg.cholesky((1.0 - c) * np.eye(cfg.rank) + c * np.ones((cfg.rank, cfg.rank)))
            G = G @ L.T
        G = G * np.exp(cfg.row_sigma * rng.standard_normal((I, 1)))
        if cfg.unit_columns:
            G = G / np.linalg.norm(G, axis=0, keepdims=True)
        out.append(G)
    return out


def _krp_rows(mats: Sequence[np.ndarray]) -> np.ndarray:
    """rows of A_last (.) ... (.) A_first in the first-index-fastest order (first matrix fastest)."""
    Z = mats[0]
    for A in mats[1:]:
        Z = (A[:, None, :] * Z[None, :, :]).reshape(-1, Z.shape[1])
    return Z


def cp_tensor(factors: Sequence[np.ndarray]) -> np.ndarray:
    """[[A]] as a flat first-index-fastest fp64 vector."""
    Z = _krp_rows(list(factors[1:]))          # J_1 x R, row j = i_2 + I_2 i_3 + ...
    X1 = factors[0] @ Z.T                     # mode-1 unfolding I_1 x J_1
    return np.ascontiguousarray(X1.T).reshape(-1)  # column-major flattening == first-index-fastest


def tensor(cfg: Config, seed: Optional[int] = None) -> np.ndarray:
    """X = [[A_true]] + rho ||X0||/||E|| E, flat first-index-fastest, in cfg.dtype."""
    s = cfg.seed if seed is None else seed
    X0 = cp_tensor(true_factors(cfg, s))
    if cfg.noise > 0.0:
        rng = np.random.default_rng([s, 2])
        E = rng.standard_normal(X0.shape[0])
        X0 = X0 + cfg.noise * (np.linalg.norm(X0) / np.linalg.norm(E)) * E
    return X0.astype(np.float64 if cfg.dtype == "f64" else np.float32)


def init_factors(cfg: Config, X: Optional[np.ndarray] = None, seed: Optional[int] = None,
                 xnorm: Optional[float] = None) -> List[np.ndarray]:
    """U[0,1] factors, norm-matched to ||X||_F (reading R13), in cfg.dtype."""
    rng = np.random.default_rng([cfg.seed if seed is None else seed, 3])
    A0 = [rng.random((I, cfg.rank)) for I in cfg.dims]
    if xnorm is None and X is not None:
        xnorm = float(np.linalg.norm(X.astype(np.float64)))
    if xnorm is not None:
        # ||[[A0]]||^2 = sum_{r,s} prod_n (A_n^T A_n)_{rs}  (Hadamard of Grams; input assembly only)
        H = np.ones((cfg.rank, cfg.rank))
        for A in A0:
            H = H * (A.T @ A)
        scale = (xnorm / math.sqrt(max(H.sum(), 1e-300))) ** (1.0 / cfg.order)
        A0 = [A * scale for A in A0]
    dt = np.float64 if cfg.dtype == "f64" else np.float32
    return [np.ascontiguousarray(A.astype(dt)) for A in A0]


# ---------------------------------------------------------------------------------------
# torch backend on a CUDA device (large configs).  Same recipe; the random stream is
# torch's, so values differ from the numpy backend.
# ---------------------------------------------------------------------------------------

def tensor_torch(cfg: Config, device="cuda", seed: Optional[int] = None, slab=None, chunk_elems: int = 1 << 28):
    """Returns (X flat torch tensor in cfg.dtype on `device`, true factors (torch fp64 on device),
    ||X||_F computed in fp64).  `slab=(k0, k1)` generates only X[..., k0:k1] (last mode), still
    first-index-fastest, with the noise scale fixed by the FULL tensor (exact ratio)."""
    import torch

    s = cfg.seed if seed is None else seed
    g = torch.Generator(device=device)
    g.manual_seed(1_000_003 * s + 11)
    A = []
    for I in cfg.dims:
        G = torch.randn((I, cfg.rank), generator=g, device=device, dtype=torch.float64)
        if cfg.congruence > 0.0:
            c = cfg.congruence
            L = torch.linalg.cholesky((1.0 - c) * torch.eye(cfg.rank, device=device, dtype=torch.float64)
                                      + c * torch.ones((cfg.rank, cfg.rank), device=device, dtype=torch.float64))
            G = G @ L.T
        G = G * torch.exp(cfg.row_sigma * torch.randn((I, 1), generator=g, device=device, dtype=torch.float64))
        if cfg.unit_columns:
            G = G / torch.linalg.norm(G, dim=0, keepdim=True)
        A.append(G)
    dims = cfg.dims
    I_last = dims[-1]
    inner = int(np.prod(dims[:-1]))
    k0, k1 = (0, I_last) if slab is None else slab
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    X = torch.empty(inner * (k1 - k0), dtype=tdt, device=device)
    # inner KRP rows (first mode fastest) of modes 1..N-2 (0-based), times A_0^T
    Zin = A[1]
    for M in A[2:-1]:
        Zin = (M[:, None, :] * Zin[None, :, :]).reshape(-1, cfg.rank)
    rows_per = max(1, chunk_elems // inner)

    def x0_rows(a, b):  # X0[..., a:b] as (b-a, inner) fp64
        Zc = (A[-1][a:b, None, :] * Zin[None, :, :]).reshape(-1, cfg.rank)   # ((b-a)*J_mid) x R
        return (Zc @ A[0].T).reshape(b - a, inner)

    def noise_rows(a, b):
        gg = torch.Generator(device=device)
        gg.manual_seed(2_000_029 * s + 17 + a)
        return torch.randn((b - a, inner), generator=gg, device=device, dtype=torch.float64)

    x0n2 = torch.zeros((), dtype=torch.float64, device=device)
    en2 = torch.zeros((), dtype=torch.float64, device=device)
    for a in range(0, I_last, rows_per):
        b = min(I_last, a + rows_per)
        x0n2 += (x0_rows(a, b) ** 2).sum()
        if cfg.noise > 0.0:
            en2 += (noise_rows(a, b) ** 2).sum()
    rho = cfg.noise * math.sqrt(x0n2.item()) / math.sqrt(en2.item()) if cfg.noise > 0.0 else 0.0
    xn2 = torch.zeros((), dtype=torch.float64, device=device)
    for a in range(0, I_last, rows_per):
        b = min(I_last, a + rows_per)
        blk = x0_rows(a, b)
        if rho:
            blk = blk + rho * noise_rows(a, b)
        lo, hi = max(a, k0), min(b, k1)
        xn2 += (blk.to(tdt).to(torch.float64) ** 2).sum()
        if lo < hi:
            X[(lo - k0) * inner:(hi - k0) * inner] = blk[lo - a:hi - a].reshape(-1).to(tdt)
    return X, A, math.sqrt(xn2.item())


def init_factors_torch(cfg: Config, xnorm: float, device="cuda", seed: Optional[int] = None):
    import torch

    s = cfg.seed if seed is None else seed
    g = torch.Generator(device=device)
    g.manual_seed(3_000_017 * s + 5)
    A0 = [torch.rand((I, cfg.rank), generator=g, device=device, dtype=torch.float64) for I in cfg.dims]
    H = torch.ones((cfg.rank, cfg.rank), dtype=torch.float64, device=device)
    for A in A0:
        H = H * (A.T @ A)
    scale = (xnorm / math.sqrt(max(H.sum().item(), 1e-300))) ** (1.0 / cfg.order)
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    return [(A * scale).to(tdt).contiguous() for A in A0]


def spread_magnitude(I: int, J: int, R: int, spread: int, magnitude: float, noise: float = 0.05,
                     seed: int = 0):
    """The paper's I x I x J experiment tensor with SPEC.md's
    stand-in for the cited spread / magnitude rule: two I x R and one J x R factors with N(0,1)
    entries, the first three columns zeroed, then in each zeroed column `spread` distinct rows
    (uniform) set to magnitude * (random sign); X = [[A]] + noise ||X0|| / ||E|| E.
    Returns (X flat first-index-fastest fp64, clean [[A]], factors)."""
    if spread > min(I, J) or R < 3:
        raise ValueError("spread exceeds a row count or R < 3")
    rng = np.random.default_rng([seed, 11])
    fs = []
    for n_rows in (I, I, J):
        A = rng.standard_normal((n_rows, R))
        A[:, :3] = 0.0
        for c in range(3):
            rows = rng.choice(n_rows, size=spread, replace=False)
            A[rows, c] = magnitude * rng.choice([-1.0, 1.0], size=spread)
        fs.append(A)
    X0 = cp_tensor(fs)
    E = rng.standard_normal(X0.shape[0])
    X = X0 + noise * (np.linalg.norm(X0) / np.linalg.norm(E)) * E if noise > 0.0 else X0.copy()
    return X, X0, fs
