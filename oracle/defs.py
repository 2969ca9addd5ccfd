"""Plain definitions (explicit constructions) for tiny inputs -- TEST INFRASTRUCTURE ONLY.

Where a sub-result of the method has a plain definition, it is written out here directly
(numpy, fp64, explicit loops or library primitives) so that tests can pin the step-by-step
oracle in ``oracle.c`` against it.  Only small tensors (J_n up to a few thousand).
"""
from __future__ import annotations

import itertools
from typing import List, Sequence

import numpy as np


def tuples(dims, n):
    """all (N-1)-tuples for mode n in eq:map order: first remaining mode fastest."""
    rest = [range(d) for k, d in enumerate(dims) if k != n]
    # itertools.product varies the LAST factor fastest; reverse to make the first fastest
    for t in itertools.product(*reversed(rest)):
        yield tuple(reversed(t))


def element(X_flat, dims, sub):
    """X[i_1..i_N] of a first-index-fastest tensor by the plain offset definition."""
    off, stride = 0, 1
    for i, d in zip(sub, dims):
        off += i * stride
        stride *= d
    return X_flat[off]


def unfold(X_flat, dims, n) -> np.ndarray:
    """explicit mode-n unfolding X_(n) (I_n x J_n), column j = j-th tuple of eq:map."""
    cols = []
    for t in tuples(dims, n):
        col = []
        for i in range(dims[n]):
            sub = list(t)
            sub.insert(n, i)
            col.append(element(X_flat, dims, sub))
        cols.append(col)
    return np.array(cols, dtype=np.float64).T


def krp(factors: Sequence[np.ndarray], n: int) -> np.ndarray:
    """Z^(n) = A^(N) (.) ... (.) A^(n+1) (.) A^(n-1) (.) ... (.) A^(1), by the
    definition of the Khatri-Rao product as the matching column-wise Kronecker product."""
    mats = [np.asarray(A, dtype=np.float64) for k, A in enumerate(factors) if k != n]
    R = mats[0].shape[1]
    cols = []
    for r in range(R):
        c = np.ones(1)
        for A in reversed(mats):     # A^(N) first (leftmost) ... A^(1) last
            c = np.kron(c, A[:, r])
        cols.append(c)
    return np.array(cols).T


def full_gradient(X_flat, dims, factors, n) -> np.ndarray:
    """g_bar = (1/J_n)(A^(n) Z^T Z - X_(n) Z)  (the quantity every estimator of eq:gradient1 /
    eq:gradient2 is unbiased for, reading R1)."""
    Z = krp(factors, n)
    Xn = unfold(X_flat, dims, n)
    Jn = Z.shape[0]
    A = np.asarray(factors[n], dtype=np.float64)
    return (A @ (Z.T @ Z) - Xn @ Z) / Jn


def objective(X_flat, dims, factors) -> float:
    """f = 1/2 ||X - [[A]]||_F^2 via the mode-1 unfolding identity
    X_(1) ~ A^(1) Z^(1)^T."""
    Z = krp(factors, 0)
    Xn = unfold(X_flat, dims, 0)
    return 0.5 * float(np.sum((Xn - np.asarray(factors[0]) @ Z.T) ** 2))


def row_prob_table(tables, dims, n) -> np.ndarray:
    """explicit J_n-vector P_j = prod_{k != n} q_k[i_k] / T_k (Lemma 2.7)."""
    P = []
    for t in tuples(dims, n):
        p = 1.0
        pos = 0
        for k in range(len(dims)):
            if k == n:
                continue
            q, T = tables[k]
            p *= float(q[t[pos]]) / float(T)
            pos += 1
        P.append(p)
    return np.array(P)


def leverage_svd(A, tol=None):
    """leverage scores from the left singular vectors (library routine), rank-truncated."""
    U, s, _ = np.linalg.svd(np.asarray(A, dtype=np.float64), full_matrices=False)
    if tol is None:
        tol = max(A.shape) * np.finfo(float).eps * (s[0] if s.size else 0.0)
    r = int(np.sum(s > tol))
    return np.sum(U[:, :r] ** 2, axis=1), r


def als_solution(X_flat, dims, factors, n) -> np.ndarray:
    """minimiser of eq:lsq_krp: A = X_(n) Z (Z^T Z)^{-1}."""
    Z = krp(factors, n)
    Xn = unfold(X_flat, dims, n)
    return np.linalg.solve(Z.T @ Z, (Xn @ Z).T).T


def windows(I, b):
    """contiguous windows of length b partitioning range(I), last one ragged (reading R6)."""
    return [list(range(s, min(I, s + b))) for s in range(0, I, b)]
