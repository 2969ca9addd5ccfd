"""CPU oracle for the importance-sampled SGD step of arXiv 2103.04081 (BrawsCPD / AdawsCPD).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_2103_04081_b200`` never imports it, and the two share no code.

``oracle/oracle.c`` holds the step-by-step algorithm (plain C, fp64, single thread, no FMA
contraction); ``oracle/defs.py`` holds the plain definitions (explicit unfolding, explicit
Khatri-Rao product, explicit J_n-row probability table, exact expectations) used to pin it.
This module is a thin ctypes binding: argument marshalling only.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")

UNIFORM, LEVERAGE, EUCLIDEAN, BLOCK_LEVERAGE, BLOCK_EUCLIDEAN = 0, 1, 2, 3, 4
STRATEGIES = {"uniform": 0, "leverage": 1, "euclidean": 2, "block_leverage": 3, "block_euclidean": 4}
STEP_FIXED, STEP_ADAPTIVE, STEP_ALS = 0, 1, 2
ORDER_CYCLIC, ORDER_RANDOM = 0, 1

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liborc.so (gcc, fp64, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i64, i32, u64, dbl = C.c_int64, C.c_int, C.c_uint64, C.c_double
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_linear_index.argtypes = [i32, P, i32, P]
        L.orc_linear_index.restype = i64
        L.orc_tensor_samp.argtypes = [i32, P, P, i32, i64, P, P]
        L.orc_skr.argtypes = [i32, P, i32, P, i32, i64, P, P]
        L.orc_leverage_scores.argtypes = [i64, i32, P, P, P]
        L.orc_row_probs.argtypes = [i32, i64, i32, P, P, P]
        L.orc_quantize.argtypes = [i32, i64, P, P, P]
        L.orc_build_table.argtypes = [i32, i64, i32, P, P, P, P]
        L.orc_default_windows.argtypes = [i32, P, i32, i64, P]
        L.orc_sample.argtypes = [i32, P, i32, i32, i64, P, P, P, u64, u64, P, P, P, P]
        L.orc_sample_stratified.argtypes = [i32, P, i32, i32, i64, P, P, u64, u64, i32, P, P, P, P]
        L.orc_gradient.argtypes = [i32, P, i32, P, P, i32, i32, i64, i64, P, P, P, P, P]
        L.orc_update_fixed.argtypes = [i64, i32, P, P, dbl]
        L.orc_update_adaptive.argtypes = [i64, i32, P, P, P, dbl, dbl, dbl]
        L.orc_update_als.argtypes = [i64, i32, P, P, P]
        L.orc_sym_pinv.argtypes = [i32, P, P]
        L.orc_fit.argtypes = [i32, P, P, i32, P, P, P, P]
        L.orc_random_mode.argtypes = [u64, u64, i32]
        L.orc_run.argtypes = [i32, P, i32, P, P, P, i32, i32, i32, i64, P, dbl, P, dbl, dbl, dbl, u64, u64, i64, P]
        L.orc_run_f32.argtypes = L.orc_run.argtypes
        L.orc_run_from.argtypes = [i32, P, i32, P, i32, P, P, i32, i32, i32, i32, i64, P, dbl, P, dbl, dbl, dbl, u64,
                                   u64, i64, P]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _chk(st: int, what: str):
    if st != 0:
        raise OracleError(f"{what}: oracle status {st}")


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dims(dims):
    return np.ascontiguousarray(dims, dtype=np.int64)


def _ptrs(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ----------------------------------------------------------------------------------------

def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def linear_index(dims, n: int, tuple_) -> int:
    d = _dims(dims)
    t = np.ascontiguousarray(tuple_, dtype=np.int32)
    j = lib().orc_linear_index(len(d), _p(d), n, _p(t))
    if j < 0:
        raise OracleError("index out of range")
    return int(j)


def tensor_samp(X: np.ndarray, dims, n: int, idx: np.ndarray) -> np.ndarray:
    """Alg. 5: returns X_(n)(:, F) as an (I_n, B) array."""
    d = _dims(dims)
    Xf = _f64(X).ravel(order="F") if X.ndim > 1 else _f64(X)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    B = idx.shape[0]
    out = np.zeros((B, d[n]), dtype=np.float64)
    _chk(lib().orc_tensor_samp(len(d), _p(d), _p(Xf), n, B, _p(idx), _p(out)), "tensor_samp")
    return out.T.copy()


def skr(factors, n: int, idx: np.ndarray) -> np.ndarray:
    fs = [_f64(A) for A in factors]
    d = _dims([A.shape[0] for A in fs])
    R = fs[0].shape[1]
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    Z = np.zeros((idx.shape[0], R), dtype=np.float64)
    _chk(lib().orc_skr(len(fs), _p(d), R, _ptrs(fs), n, idx.shape[0], _p(idx), _p(Z)), "skr")
    return Z


def leverage_scores(A: np.ndarray):
    A = _f64(A)
    ell = np.zeros(A.shape[0])
    rank = C.c_int(0)
    _chk(lib().orc_leverage_scores(A.shape[0], A.shape[1], _p(A), _p(ell), C.byref(rank)), "leverage")
    return ell, rank.value


def row_probs(strategy: int, A: np.ndarray) -> np.ndarray:
    A = _f64(A)
    p = np.zeros(A.shape[0])
    _chk(lib().orc_row_probs(strategy, A.shape[0], A.shape[1], _p(A), _p(p), None), "row_probs")
    return p


def quantize(strategy: int, p: np.ndarray):
    p = _f64(p)
    q = np.zeros(p.shape[0], dtype=np.uint64)
    T = C.c_uint64(0)
    _chk(lib().orc_quantize(strategy, p.shape[0], _p(p), _p(q), C.byref(T)), "quantize")
    return q, int(T.value)


def build_table(strategy: int, A: np.ndarray):
    """returns (p fp64, q uint64, T)"""
    A = _f64(A)
    p = np.zeros(A.shape[0])
    q = np.zeros(A.shape[0], dtype=np.uint64)
    T = C.c_uint64(0)
    _chk(lib().orc_build_table(strategy, A.shape[0], A.shape[1], _p(A), _p(p), _p(q), C.byref(T)), "table")
    return p, q, int(T.value)


def default_windows(dims, n: int, B: int) -> np.ndarray:
    d = _dims(dims)
    w = np.zeros(len(d) - 1, dtype=np.int32)
    lib().orc_default_windows(len(d), _p(d), n, B, _p(w))
    return w


def sample(dims, n: int, strategy: int, B: int, tables, seed: int, it: int, window=None):
    """tables: list of (q, T) per mode (entry n ignored).  Returns idx (B_eff, N-1) int32,
    w (B_eff,) fp64 weights, pj (B_eff,) probabilities."""
    d = _dims(dims)
    N = len(d)
    qs = [np.ascontiguousarray(t[0], dtype=np.uint64) for t in tables]
    T = np.ascontiguousarray([t[1] for t in tables], dtype=np.uint64)
    win = None if window is None else np.ascontiguousarray(window, dtype=np.int32)
    Bmax = B if win is None else max(B, int(np.prod(win)))
    idx = np.zeros((Bmax, N - 1), dtype=np.int32)
    w = np.zeros(Bmax)
    pj = np.zeros(Bmax)
    Beff = C.c_int64(0)
    _chk(lib().orc_sample(N, _p(d), n, strategy, B, None if win is None else _p(win), _ptrs(qs), _p(T),
                          C.c_uint64(seed), C.c_uint64(it), _p(idx), _p(w), _p(pj), C.byref(Beff)), "sample")
    b = Beff.value
    return idx[:b].copy(), w[:b].copy(), pj[:b].copy()


def sample_stratified(dims, n: int, strategy: int, B: int, tables, seed: int, it: int, slab_lo):
    """stratified per-slab draws (orc_sample_stratified; reading R26).  slab_lo: P+1 slab bounds of the
    last mode.  Returns idx (B, N-1) int32, w (B,) fp64, pj (B,) with 1/(B J_n pj) = w."""
    d = _dims(dims)
    N = len(d)
    qs = [np.ascontiguousarray(t[0], dtype=np.uint64) for t in tables]
    T = np.ascontiguousarray([t[1] for t in tables], dtype=np.uint64)
    lo = np.ascontiguousarray(slab_lo, dtype=np.int64)
    idx = np.zeros((B, N - 1), dtype=np.int32)
    w = np.zeros(B)
    pj = np.zeros(B)
    _chk(lib().orc_sample_stratified(N, _p(d), n, strategy, B, _ptrs(qs), _p(T), C.c_uint64(seed), C.c_uint64(it),
                                     len(lo) - 1, _p(lo), _p(idx), _p(w), _p(pj)), "sample_stratified")
    return idx, w, pj


def gradient(X: np.ndarray, dims, factors, n: int, strategy: int, B: int, idx, pj):
    """eq:gradient1 / eq:gradient2.  Returns (G, Gamma, M)."""
    d = _dims(dims)
    fs = [_f64(A) for A in factors]
    R = fs[0].shape[1]
    Xf = _f64(X).ravel(order="F") if X.ndim > 1 else _f64(X)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    pj = _f64(pj)
    In = int(d[n])
    G = np.zeros((In, R)); Gam = np.zeros((R, R)); M = np.zeros((In, R))
    _chk(lib().orc_gradient(len(d), _p(d), R, _p(Xf), _ptrs(fs), n, strategy, B, idx.shape[0], _p(idx), _p(pj),
                            _p(G), _p(Gam), _p(M)), "gradient")
    return G, Gam, M


def update_fixed(A: np.ndarray, G: np.ndarray, alpha: float) -> np.ndarray:
    A = _f64(A).copy()
    G = _f64(G)
    lib().orc_update_fixed(A.shape[0], A.shape[1], _p(A), _p(G), alpha)
    return A


def sym_pinv(Gam: np.ndarray):
    """Gamma^+ on the numerically full-rank pivot set (natural-order sweep, tol R eps max diag).
    Returns (W, rank)."""
    G = _f64(Gam)
    W = np.zeros_like(G)
    rk = lib().orc_sym_pinv(G.shape[0], _p(G), _p(W))
    if rk < 0:
        raise OracleError("sym_pinv: out of memory")
    return W, int(rk)


def update_als(M: np.ndarray, Gam: np.ndarray) -> np.ndarray:
    """the sampled least-squares step A = M Gamma^+ (eq:lsq_krp on eq:gradient1/2's M, Gamma)."""
    M = _f64(M)
    G = _f64(Gam)
    A = np.zeros_like(M)
    _chk(lib().orc_update_als(M.shape[0], M.shape[1], _p(A), _p(M), _p(G)), "update_als")
    return A


def update_adaptive(A, S, G, eta, b=0.0, eps=0.0):
    A = _f64(A).copy(); S = _f64(S).copy(); G = _f64(G)
    lib().orc_update_adaptive(A.shape[0], A.shape[1], _p(A), _p(S), _p(G), eta, b, eps)
    return A, S


def fit(X: np.ndarray, factors) -> float:
    fs = [_f64(A) for A in factors]
    d = _dims([A.shape[0] for A in fs])
    Xf = _f64(X).ravel(order="F") if X.ndim > 1 else _f64(X)
    out = C.c_double(0.0)
    _chk(lib().orc_fit(len(d), _p(d), _p(Xf), fs[0].shape[1], _ptrs(fs), C.byref(out), None, None), "fit")
    return out.value


def random_mode(seed: int, it: int, N: int) -> int:
    return int(lib().orc_random_mode(C.c_uint64(seed), C.c_uint64(it), N))


def run(X, factors, strategy: int, rule: int, B: int, iters: int, *, order=ORDER_CYCLIC, window=None,
        alpha=0.0, alphas=None, eta=0.1, b=0.0, eps=0.0, seed=0, r0=0, S=None, first_mode=0):
    """Alg. 6 / Alg. 7 for `iters` iterations.  Returns (factors, S, modes); inputs are copied."""
    fs = [_f64(A).copy() for A in factors]
    d = _dims([A.shape[0] for A in fs])
    N = len(fs)
    R = fs[0].shape[1]
    Ss = [np.zeros_like(A) for A in fs] if S is None else [_f64(s).copy() for s in S]
    x32 = X.dtype == np.float32 and X.ndim == 1 and X.flags["C_CONTIGUOUS"]
    # an fp32 flat tensor is read in place by the fp32 entry (no fp64 copy of a 32 GB tensor)
    Xf = X if x32 else (_f64(X).ravel(order="F") if X.ndim > 1 else _f64(X))
    win = None if window is None else np.ascontiguousarray(window, dtype=np.int32)
    al = None if alphas is None else _f64(alphas)
    modes = np.zeros(max(iters, 1), dtype=np.int32)
    _chk(lib().orc_run_from(N, _p(d), R, _p(Xf), 1 if x32 else 0, _ptrs(fs), _ptrs(Ss), strategy, rule, order,
                            int(first_mode), B,
                       None if win is None else _p(win), alpha, None if al is None else _p(al), eta, b, eps,
                       C.c_uint64(seed), C.c_uint64(r0), iters, _p(modes)), "run")
    return fs, Ss, modes[:iters]
