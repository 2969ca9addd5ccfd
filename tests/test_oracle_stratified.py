"""Pins of the stratified per-slab sampler (oracle.sample_stratified, reading R26), CPU.

The sampler splits the batch into P strata, one per contiguous slab of the LAST mode, and draws stratum
g's last-mode index from the slab's conditional law.  What fixes it (R26):
  * special cases: P = 1, and the update of the last mode itself (its fibers span every slab), are the
    unstratified sampler of eq:ik bit for bit;
  * the same Philox counters: every other position of every row equals the unstratified draw;
  * the law: stratum g's fibers follow the explicit J_n table P_j (Lemma 2.7)
    conditioned on i_last in slab g (chi^2), and the returned pj equals (B_g/B) P_j / mass_g computed
    from that explicit table;
  * unbiasedness (Theorem 5.1, stratum by stratum): with one row per stratum the
    exact expectation over the design, sum_g sum_{j in g} (P_j / mass_g) G({j}), equals the full
    gradient g_bar of defs.full_gradient -- also with a zero-mass slab, where it equals the
    unstratified sampler's exact expectation;
  * a Monte-Carlo mean of the stratified estimator over many iterations approaches g_bar.
"""
import numpy as np
import pytest
import scipy.stats

import oracle as orc
from oracle import defs

ROWWISE = ["uniform", "leverage", "euclidean"]


def rand_factors(dims, R, seed=0, row_sigma=0.5):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((I, R)) * np.exp(row_sigma * rng.standard_normal((I, 1))) for I in dims]


def rand_tensor(dims, seed=1):
    return np.random.default_rng(seed).standard_normal(int(np.prod(dims)))


def tables_for(strategy, factors):
    st = orc.STRATEGIES[strategy]
    return [orc.build_table(st, A)[1:] for A in factors]


def strata(B, P):
    out, off = [], 0
    for g in range(P):
        bg = B // P + (1 if g < B % P else 0)
        out.append((off, off + bg))
        off += bg
    return out


@pytest.mark.parametrize("strategy", ROWWISE)
def test_special_cases_equal_unstratified(strategy):
    dims = (5, 6, 8)
    fs = rand_factors(dims, 3, seed=1)
    tabs = tables_for(strategy, fs)
    st = orc.STRATEGIES[strategy]
    for n in range(3):
        a = orc.sample(dims, n, st, 40, tabs, 7, 3)
        b = orc.sample_stratified(dims, n, st, 40, tabs, 7, 3, [0, 8])  # P = 1
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
    a = orc.sample(dims, 2, st, 40, tabs, 7, 3)  # the last mode: no strata, whatever P
    b = orc.sample_stratified(dims, 2, st, 40, tabs, 7, 3, [0, 3, 5, 8])
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("strategy", ROWWISE)
def test_same_counters_and_slab_membership(strategy):
    dims = (5, 6, 9)
    fs = rand_factors(dims, 3, seed=2)
    tabs = tables_for(strategy, fs)
    st = orc.STRATEGIES[strategy]
    lo = [0, 2, 5, 9]
    for n in (0, 1):
        B = 31
        a, _, _ = orc.sample(dims, n, st, B, tabs, 11, 5)
        b, w, pj = orc.sample_stratified(dims, n, st, B, tabs, 11, 5, lo)
        assert np.array_equal(a[:, 0], b[:, 0])  # the other remaining mode: the same draw
        for g, (b0, b1) in enumerate(strata(B, 3)):
            assert np.all((b[b0:b1, 1] >= lo[g]) & (b[b0:b1, 1] < lo[g + 1]))
        assert np.all(w > 0)
    with pytest.raises(orc.OracleError):
        orc.sample_stratified(dims, 0, st, 2, tabs, 11, 5, lo)  # B < P
    with pytest.raises(orc.OracleError):
        orc.sample_stratified(dims, 0, orc.BLOCK_LEVERAGE, 8, tabs, 11, 5, lo)


@pytest.mark.parametrize("strategy", ROWWISE)
def test_stratum_law_chi_square_and_pj(strategy):
    """stratum g's fibers ~ P_j | i_last in slab g (Pearson chi^2 of 60k draws per stratum, p > 1e-4);
    every returned pj = (B_g/B) P_j / mass_g and w = 1/(B J_n pj)"""
    dims = (3, 4, 6)
    n = 0
    fs = rand_factors(dims, 2, seed=8, row_sigma=0.4)
    tabs = tables_for(strategy, fs)
    st = orc.STRATEGIES[strategy]
    lo = [0, 2, 6]
    P = defs.row_prob_table(tabs, dims, n)  # j = i_1 + 4 i_2 (eq:map order)
    B = 120_000
    idx, w, pj = orc.sample_stratified(dims, n, st, B, tabs, 21, 0, lo)
    j = idx[:, 0].astype(np.int64) + 4 * idx[:, 1].astype(np.int64)
    Jn = 4 * 6
    for g, (b0, b1) in enumerate(strata(B, 2)):
        inslab = np.array([lo[g] <= jj // 4 < lo[g + 1] for jj in range(Jn)])
        mass = P[inslab].sum()
        law = np.where(inslab, P / mass, 0.0)
        obs = np.bincount(j[b0:b1], minlength=Jn)[inslab]
        exp = law[inslab] * (b1 - b0)
        assert exp.min() >= 5
        chi2 = float(((obs - exp) ** 2 / exp).sum())
        assert scipy.stats.chi2.sf(chi2, int(inslab.sum()) - 1) > 1e-4
        ref = ((b1 - b0) / B) * law[j[b0:b1]]
        np.testing.assert_allclose(pj[b0:b1], ref, rtol=1e-14)
    np.testing.assert_allclose(w, 1.0 / (B * Jn * pj), rtol=1e-14)


def _exact_expectation(X, dims, fs, n, strategy, tabs, lo):
    """sum over strata g and fibers j of slab g: (P_j / mass_g) G({j}) with B = P rows (one per stratum),
    G from orc.gradient with pj = (1/P) P_j / mass_g -- the stratified estimator's exact mean"""
    st = orc.STRATEGIES[strategy]
    Pn = defs.row_prob_table(tabs, dims, n)
    tup = list(defs.tuples(dims, n))
    nP = len(lo) - 1
    E = np.zeros((dims[n], fs[0].shape[1]))
    for g in range(nP):
        members = [jj for jj, t in enumerate(tup) if lo[g] <= t[-1] < lo[g + 1]]
        mass = sum(Pn[jj] for jj in members)
        if mass == 0.0:
            continue
        for jj in members:
            if Pn[jj] == 0.0:
                continue
            pc = Pn[jj] / mass
            G, _, _ = orc.gradient(X, dims, fs, n, st, nP, np.array([tup[jj]], dtype=np.int32),
                                   np.array([pc / nP]))
            E += pc * G
    return E


@pytest.mark.parametrize("strategy", ROWWISE)
def test_exact_expectation_is_full_gradient(strategy):
    dims = (3, 4, 5)
    fs = rand_factors(dims, 2, seed=3)
    X = rand_tensor(dims, seed=4)
    tabs = tables_for(strategy, fs)
    for n in (0, 1):
        for lo in ([0, 2, 5], [0, 1, 3, 4, 5]):
            E = _exact_expectation(X, dims, fs, n, strategy, tabs, lo)
            np.testing.assert_allclose(E, defs.full_gradient(X, dims, fs, n), rtol=1e-12, atol=1e-14)


def test_zero_mass_slab():
    """a slab whose last-mode rows are all zero: its stratum's rows carry w = 0 (pj = inf), and the
    exact expectation equals the unstratified sampler's (both see only the probability-positive fibers)"""
    dims = (3, 4, 6)
    fs = rand_factors(dims, 2, seed=5)
    fs[2][2:4] = 0.0  # slab [2, 4) of the last mode has zero Euclidean / leverage mass
    X = rand_tensor(dims, seed=6)
    tabs = tables_for("euclidean", fs)
    lo = [0, 2, 4, 6]
    idx, w, pj = orc.sample_stratified(dims, 0, orc.EUCLIDEAN, 9, tabs, 3, 1, lo)
    assert np.all(w[3:6] == 0.0) and np.all(np.isinf(pj[3:6])) and np.all(idx[3:6, 1] == 2)
    assert np.all(w[:3] > 0) and np.all(w[6:] > 0)
    G, _, _ = orc.gradient(X, dims, fs, 0, orc.EUCLIDEAN, 9, idx, pj)
    assert np.all(np.isfinite(G))
    E = _exact_expectation(X, dims, fs, 0, "euclidean", tabs, lo)
    Pn = defs.row_prob_table(tabs, dims, 0)
    E1 = np.zeros_like(E)
    for jj, t in enumerate(defs.tuples(dims, 0)):
        if Pn[jj] > 0:
            G1, _, _ = orc.gradient(X, dims, fs, 0, orc.EUCLIDEAN, 1, np.array([t], dtype=np.int32), np.array([Pn[jj]]))
            E1 += Pn[jj] * G1
    np.testing.assert_allclose(E, E1, rtol=1e-12, atol=1e-14)


def test_monte_carlo_mean_approaches_full_gradient():
    """mean of the stratified estimator over 4000 iterations (B = 64, P = 4 slabs) within 2 % of g_bar"""
    dims = (6, 5, 16)
    fs = rand_factors(dims, 3, seed=9)
    X = rand_tensor(dims, seed=10)
    tabs = tables_for("leverage", fs)
    lo = [0, 3, 8, 12, 16]
    acc = np.zeros((dims[0], 3))
    its = 4000
    for it in range(its):
        idx, _, pj = orc.sample_stratified(dims, 0, orc.LEVERAGE, 64, tabs, 17, it, lo)
        G, _, _ = orc.gradient(X, dims, fs, 0, orc.LEVERAGE, 64, idx, pj)
        acc += G
    gbar = defs.full_gradient(X, dims, fs, 0)
    assert np.linalg.norm(acc / its - gbar) <= 0.02 * np.linalg.norm(gbar)
