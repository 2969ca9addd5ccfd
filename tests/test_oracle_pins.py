"""Pins of the CPU oracle against what the paper and the mathematics fix (CPU only).

Each test pins one oracle function to something other than itself: a published known-answer
vector, a closed form, an invariant, a special case that reduces to a library routine, or
brute force on tiny inputs (exhaustive enumeration).  Citations: PAPER.md:<lines> (<label>),
SPEC.md:<lines> for the worked examples of the written-from-the-paper spec.
"""
import itertools
import math
import os

import numpy as np
import pytest
import scipy.linalg
import scipy.stats

from oracle import defs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
S = ["uniform", "leverage", "euclidean", "block_leverage", "block_euclidean"]
ROWWISE = ["uniform", "leverage", "euclidean"]
BLOCK = ["block_leverage", "block_euclidean"]


def rand_factors(dims, R, seed=0, row_sigma=0.5):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((I, R)) * np.exp(row_sigma * rng.standard_normal((I, 1))) for I in dims]


def rand_tensor(dims, seed=1):
    return np.random.default_rng(seed).standard_normal(int(np.prod(dims)))


def tables_for(orc, strategy, factors):
    st = orc.STRATEGIES[strategy]
    out = []
    for A in factors:
        p, q, T = orc.build_table(st, A)
        out.append((q, T))
    return out


# ---------------------------------------------------------------------------------------- Philox
def test_philox_known_answers(orc):
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        assert orc.philox(w[0:4], w[4:6]).tolist() == w[6:10]
        n += 1
    assert n == 3


# ---------------------------------------------------------------------------------------- index map
def test_linear_index_spec_examples(orc):
    """SPEC.md:51-53 worked values (1-based there): dims (2,3,4)."""
    assert orc.linear_index((2, 3, 4), 0, (0, 0)) == 0      # (i2,i3)=(1,1) -> j=1
    assert orc.linear_index((2, 3, 4), 0, (2, 3)) == 11     # (3,4) -> j=12
    assert orc.linear_index((2, 3, 4), 1, (1, 0)) == 1      # mode 2, (i1,i3)=(2,1) -> j=2


@pytest.mark.parametrize("seed", range(6))
def test_linear_index_bijection(orc, seed):
    """eq:map is a bijection onto [0, J_n) and enumerates tuples in
    first-remaining-fastest order (brute force, N <= 4, I <= 6)."""
    rng = np.random.default_rng(seed)
    N = int(rng.integers(3, 5))
    dims = tuple(int(x) for x in rng.integers(1, 7, size=N))
    for n in range(N):
        js = [orc.linear_index(dims, n, t) for t in defs.tuples(dims, n)]
        assert js == list(range(int(np.prod(dims) // dims[n])))


def test_linear_index_out_of_range(orc):
    with pytest.raises(orc.OracleError):
        orc.linear_index((2, 3, 4), 0, (3, 0))


# ---------------------------------------------------------------------------------------- fibers
def test_tensor_samp_spec_example(orc):
    """2x2x2 tensor with values 1..8 first-index-fastest, mode 1, tuple (1,1) ->
    column (1,2)."""
    X = np.arange(1, 9, dtype=np.float64)
    out = orc.tensor_samp(X, (2, 2, 2), 0, np.array([[0, 0]]))
    assert out[:, 0].tolist() == [1.0, 2.0]


@pytest.mark.parametrize("dims", [(3, 4, 5), (2, 3, 2, 4), (5, 1, 3)])
def test_tensor_samp_reproduces_unfolding(orc, dims):
    """exhaustive ordered tuple set reproduces the explicitly built X_(n)."""
    X = rand_tensor(dims)
    for n in range(len(dims)):
        idx = np.array(list(defs.tuples(dims, n)), dtype=np.int32)
        got = orc.tensor_samp(X, dims, n, idx)
        assert np.array_equal(got, defs.unfold(X, dims, n))


# ---------------------------------------------------------------------------------------- SKR
@pytest.mark.parametrize("dims", [(3, 4, 5), (2, 3, 2, 4)])
def test_skr_matches_explicit_krp_and_scipy(orc, dims):
    """Alg. 1 rows == rows of the explicit KRP == scipy.linalg.khatri_rao
    applied as A^(N) (.) ... (.) A^(1)."""
    fs = rand_factors(dims, 3)
    for n in range(len(dims)):
        idx = np.array(list(defs.tuples(dims, n)), dtype=np.int32)
        Z = orc.skr(fs, n, idx)
        Zdef = defs.krp(fs, n)
        mats = [A for k, A in enumerate(fs) if k != n]
        Zsp = mats[-1]
        for A in reversed(mats[:-1]):
            Zsp = scipy.linalg.khatri_rao(Zsp, A)
        np.testing.assert_allclose(Z, Zdef, rtol=1e-15, atol=0)
        np.testing.assert_allclose(Z, Zsp, rtol=1e-15, atol=0)


def test_skr_spec_example(orc):
    """mode 1 of a 3-way model, tuple picks rows; z = a2(i2,:) * a3(i3,:)."""
    A1 = np.ones((2, 2)); A2 = np.array([[1., 2.], [3., 4.]]); A3 = np.array([[5., 6.], [7., 8.], [9., 10.], [11., 12.]])
    Z = orc.skr([A1, A2, A3], 0, np.array([[0, 3]], dtype=np.int32))
    assert Z.tolist() == [[11.0, 24.0]]


# ---------------------------------------------------------------------------------------- leverage
def test_leverage_spec_example(orc):
    """[[1,0],[1,0],[0,1]] -> (0.5, 0.5, 1.0)."""
    ell, r = orc.leverage_scores(np.array([[1., 0.], [1., 0.], [0., 1.]]))
    np.testing.assert_allclose(ell, [0.5, 0.5, 1.0], rtol=0, atol=1e-15)
    assert r == 2


def test_leverage_identity_and_zero_row(orc):
    ell, r = orc.leverage_scores(np.vstack([np.eye(4), np.zeros((1, 4))]))
    np.testing.assert_allclose(ell, [1, 1, 1, 1, 0], atol=1e-15)
    assert r == 4


@pytest.mark.parametrize("shape", [(60, 5), (400, 20), (37, 9), (10, 10)])
def test_leverage_vs_svd(orc, shape):
    """Def. 2.3: any orthonormal basis gives the same scores -> equals the
    SVD basis (library routine); sum = rank; each in [0,1]."""
    rng = np.random.default_rng(shape[0])
    A = rng.standard_normal(shape) * np.exp(1.5 * rng.standard_normal((shape[0], 1)))
    ell, r = orc.leverage_scores(A)
    ref, rr = defs.leverage_svd(A)
    assert r == rr == shape[1]
    np.testing.assert_allclose(ell, ref, rtol=1e-10, atol=1e-14)
    assert abs(ell.sum() - r) < 1e-12
    assert ell.min() >= 0 and ell.max() <= 1 + 1e-12


def test_leverage_orthonormal_columns(orc):
    """A with orthonormal columns is its own Q: l_i = ||A(i,:)||^2."""
    Q, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((50, 6)))
    ell, _ = orc.leverage_scores(Q)
    np.testing.assert_allclose(ell, np.sum(Q ** 2, axis=1), rtol=1e-12, atol=1e-15)


def test_leverage_rank_deficient(orc):
    """duplicate column -> rank R-1; scores equal the rank-truncated SVD scores (reading R4)."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((30, 4))
    A[:, 3] = 2.0 * A[:, 1]
    ell, r = orc.leverage_scores(A)
    ref, rr = defs.leverage_svd(A)
    assert r == rr == 3
    np.testing.assert_allclose(ell, ref, rtol=1e-10, atol=1e-13)


def test_lemma_2_6_krp_leverage_bound(orc):
    """Lemma 2.6: l_j(Z) <= prod_k l_{i_k}(A^(k)), also for I_k > R (R5)."""
    dims = (5, 6, 7)
    fs = rand_factors(dims, 3, seed=9)
    for n in range(3):
        Z = defs.krp(fs, n)
        lz, _ = defs.leverage_svd(Z)
        per = [orc.leverage_scores(A)[0] for k, A in enumerate(fs) if k != n]
        bound = np.array([np.prod([per[p][t[p]] for p in range(2)]) for t in defs.tuples(dims, n)])
        assert np.all(lz <= bound * (1 + 1e-10) + 1e-14)
        # sum_j prod_k l/R^{N-1} = 1 for full-rank factors
        assert abs(bound.sum() / 3 ** 2 - 1.0) < 1e-12


# ---------------------------------------------------------------------------------------- probabilities
def test_euclidean_spec_example(orc):
    """rows (1,0),(0,1),(1,1) -> (0.25, 0.25, 0.5) (Def. 2.5)."""
    p = orc.row_probs(orc.EUCLIDEAN, np.array([[1., 0.], [0., 1.], [1., 1.]]))
    assert p.tolist() == [0.25, 0.25, 0.5]


def test_leverage_probs_are_ell_over_rank(orc):
    """PAPER.md:271 p_k = l(A^(k))/R; identity -> uniform 1/R."""
    p = orc.row_probs(orc.LEVERAGE, np.eye(4))
    np.testing.assert_allclose(p, 0.25, atol=1e-15)


def test_quantize_closed_form(orc):
    """contract step 3: q = rint(p 2^32) (half to even), zero stays zero, tiny positive -> 1."""
    p = np.array([0.5, 0.25, 0.0, 2.0 ** -40, (3.5) / 2 ** 32, (4.5) / 2 ** 32])
    q, T = orc.quantize(orc.LEVERAGE, p)
    assert q.tolist() == [2 ** 31, 2 ** 30, 0, 1, 4, 4]
    assert T == int(q.sum())
    qu, Tu = orc.quantize(orc.UNIFORM, np.full(7, 1 / 7))
    assert qu.tolist() == [1] * 7 and Tu == 7


def test_degenerate_tables(orc):
    with pytest.raises(orc.OracleError):
        orc.build_table(orc.EUCLIDEAN, np.zeros((5, 3)))
    with pytest.raises(orc.OracleError):
        orc.build_table(orc.LEVERAGE, np.zeros((5, 3)))


@pytest.mark.parametrize("strategy", ["leverage", "euclidean", "uniform"])
def test_product_law_sums_to_one(orc, strategy):
    """Lemma 2.7: the explicit J_n table sums to 1; in integers
    sum_j prod_k q_k = prod_k T_k exactly."""
    dims = (4, 5, 3)
    fs = rand_factors(dims, 2, seed=4)
    tabs = tables_for(orc, strategy, fs)
    for n in range(3):
        P = defs.row_prob_table(tabs, dims, n)
        assert abs(P.sum() - 1.0) < 1e-14
        qs = [tabs[k][0].astype(object) for k in range(3) if k != n]
        Ts = [tabs[k][1] for k in range(3) if k != n]
        assert sum(a * b for a in qs[0] for b in qs[1]) == Ts[0] * Ts[1]


# ---------------------------------------------------------------------------------------- sampler
def test_default_windows(orc):
    """reading R6 on the BASELINE configs."""
    assert orc.default_windows((60, 60, 60), 0, 64).tolist() == [8, 8]
    assert orc.default_windows((400, 400, 400), 1, 512).tolist() == [32, 16]
    assert orc.default_windows((100,) * 4, 2, 1024).tolist() == [16, 8, 8]
    assert orc.default_windows((2000,) * 3, 0, 4096).tolist() == [64, 64]
    assert orc.default_windows((4000,) * 3, 2, 8192).tolist() == [128, 64]
    assert orc.default_windows((5, 7, 6), 0, 64).tolist() == [7, 6]  # clamped to I_k


def test_uniform_weights_exact(orc):
    """uniform: omega = 1/B exactly (BrasCPD, PAPER.md:155 with p = 1/J_n, reading R1)."""
    dims = (7, 9, 11)
    tabs = tables_for(orc, "uniform", rand_factors(dims, 2))
    idx, w, pj = orc.sample(dims, 1, orc.UNIFORM, 37, tabs, seed=3, it=5)
    assert np.all(w == 1.0 / 37)
    assert idx.shape == (37, 2) and idx[:, 0].max() < 7 and idx[:, 1].max() < 11


def test_sampler_weights_are_exact_rationals(orc):
    """omega_b = 1/(B prod_k I_k q_k/T_k) with the contract's operation order (step 7)."""
    dims = (6, 5, 7)
    fs = rand_factors(dims, 3, seed=2)
    for strategy in ["leverage", "euclidean"]:
        tabs = tables_for(orc, strategy, fs)
        idx, w, pj = orc.sample(dims, 2, orc.STRATEGIES[strategy], 50, tabs, seed=11, it=2)
        for b in range(50):
            p0 = float(6 * int(tabs[0][0][idx[b, 0]])) / float(tabs[0][1])
            p1 = float(5 * int(tabs[1][0][idx[b, 1]])) / float(tabs[1][1])
            assert w[b] == 1.0 / (50.0 * (p0 * p1))
            P = defs.row_prob_table(tabs, dims, 2)
            assert abs(pj[b] - P[orc.linear_index(dims, 2, idx[b])]) <= 1e-16


def test_block_single_window_is_full_batch(orc):
    """block with one window per mode (b_k = I_k): p_S = 1, omega = 1/J_n, batch = all tuples."""
    dims = (4, 3, 5)
    fs = rand_factors(dims, 2)
    for strategy in BLOCK:
        tabs = tables_for(orc, strategy, fs)
        idx, w, pj = orc.sample(dims, 0, orc.STRATEGIES[strategy], 15, tabs, seed=0, it=0, window=[3, 5])
        assert idx.tolist() == [list(t) for t in defs.tuples(dims, 0)]
        assert np.all(pj == 1.0) and np.all(w == 1.0 / 15)


def test_sampler_reproducible_and_iteration_dependent(orc):
    dims = (9, 8, 7)
    tabs = tables_for(orc, "leverage", rand_factors(dims, 3))
    a = orc.sample(dims, 0, orc.LEVERAGE, 64, tabs, seed=1, it=3)
    b = orc.sample(dims, 0, orc.LEVERAGE, 64, tabs, seed=1, it=3)
    c = orc.sample(dims, 0, orc.LEVERAGE, 64, tabs, seed=1, it=4)
    assert np.array_equal(a[0], b[0]) and not np.array_equal(a[0], c[0])


@pytest.mark.parametrize("strategy", ROWWISE)
def test_sampler_law_chi_square(orc, strategy):
    """Pearson chi^2 of 200k draws vs the explicit J_n table;
    fixed seed -> deterministic; accept at p > 1e-4."""
    dims = (3, 4, 5)
    fs = rand_factors(dims, 2, seed=8, row_sigma=0.3)
    tabs = tables_for(orc, strategy, fs)
    n = 1
    B = 200_000
    idx, _, _ = orc.sample(dims, n, orc.STRATEGIES[strategy], B, tabs, seed=21, it=0)
    J = 3 * 5
    j = idx[:, 0].astype(np.int64) + 3 * idx[:, 1].astype(np.int64)
    obs = np.bincount(j, minlength=J)
    P = defs.row_prob_table(tabs, dims, n)
    exp = P * B
    assert exp.min() >= 5
    chi2 = float(((obs - exp) ** 2 / exp).sum())
    assert scipy.stats.chi2.sf(chi2, J - 1) > 1e-4


@pytest.mark.parametrize("strategy", BLOCK)
def test_block_window_law_chi_square(orc, strategy):
    """joint law of the per-mode window draws = product of window masses (eq:bik, R2)."""
    dims = (7, 6, 5)
    fs = rand_factors(dims, 2, seed=12, row_sigma=1.0)
    tabs = tables_for(orc, strategy, fs)
    n = 2
    win = [3, 2]
    D = [3, 3]
    K = 20000
    counts = np.zeros((3, 3))
    for it in range(K):
        idx, _, _ = orc.sample(dims, n, orc.STRATEGIES[strategy], 6, tabs, seed=5, it=it, window=win)
        counts[idx[0, 0] // 3, idx[0, 1] // 2] += 1
    P = np.zeros((3, 3))
    for a, wa in enumerate(defs.windows(7, 3)):
        for b, wb in enumerate(defs.windows(6, 2)):
            P[a, b] = (sum(int(tabs[0][0][i]) for i in wa) / tabs[0][1]) * (sum(int(tabs[1][0][i]) for i in wb) / tabs[1][1])
    exp = P * K
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    assert scipy.stats.chi2.sf(chi2, 8) > 1e-4


# ---------------------------------------------------------------------------------------- gradient
def test_full_gradient_finite_differences():
    """g_bar = grad(f)/J_n (reading R1) by central differences, h = 1e-6."""
    dims = (3, 4, 2)
    fs = rand_factors(dims, 2, seed=1)
    X = rand_tensor(dims, seed=2)
    for n in range(3):
        g = defs.full_gradient(X, dims, fs, n)
        Jn = np.prod(dims) // dims[n]
        fd = np.zeros_like(g)
        h = 1e-6
        for i in range(dims[n]):
            for r in range(2):
                fp = [A.copy() for A in fs]; fm = [A.copy() for A in fs]
                fp[n][i, r] += h; fm[n][i, r] -= h
                fd[i, r] = (defs.objective(X, dims, fp) - defs.objective(X, dims, fm)) / (2 * h) / Jn
        np.testing.assert_allclose(g, fd, rtol=1e-6, atol=1e-8)


def test_hadamard_of_grams_identity():
    """Z^T Z = (*)_k A^(k)T A^(k) (standard KRP identity)."""
    fs = rand_factors((3, 4, 5, 2), 3, seed=6)
    for n in range(4):
        Z = defs.krp(fs, n)
        H = np.ones((3, 3))
        for k, A in enumerate(fs):
            if k != n:
                H *= A.T @ A
        np.testing.assert_allclose(Z.T @ Z, H, rtol=1e-12)


@pytest.mark.parametrize("strategy", ROWWISE)
def test_rowwise_gradient_exact_expectation(orc, strategy):
    """Theorem 5.1 by exhaustive enumeration: sum_j P_j G({j}) = g_bar
    for eq:gradient1 with B = 1, every mode."""
    dims = (3, 4, 5)
    fs = rand_factors(dims, 2, seed=3)
    X = rand_tensor(dims, seed=4)
    tabs = tables_for(orc, strategy, fs)
    st = orc.STRATEGIES[strategy]
    for n in range(3):
        P = defs.row_prob_table(tabs, dims, n)
        E = np.zeros((dims[n], 2))
        for j, t in enumerate(defs.tuples(dims, n)):
            G, _, _ = orc.gradient(X, dims, fs, n, st, 1, np.array([t], dtype=np.int32), np.array([P[j]]))
            E += P[j] * G
        np.testing.assert_allclose(E, defs.full_gradient(X, dims, fs, n), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("strategy", BLOCK)
def test_block_gradient_exact_expectation(orc, strategy):
    """Theorem 5.1 for eq:gradient2 under reading R2 (Cartesian windows,
    ragged last window): sum_S p_S G(S) = g_bar, every mode."""
    dims = (5, 7, 6)
    fs = rand_factors(dims, 2, seed=5)
    X = rand_tensor(dims, seed=6)
    tabs = tables_for(orc, strategy, fs)
    st = orc.STRATEGIES[strategy]
    win_len = (3, 2)
    for n in range(3):
        rest = [k for k in range(3) if k != n]
        W = [defs.windows(dims[k], win_len[p]) for p, k in enumerate(rest)]
        E = np.zeros((dims[n], 2))
        tot = 0.0
        for wa in W[0]:
            for wb in W[1]:
                pS = (sum(int(tabs[rest[0]][0][i]) for i in wa) / tabs[rest[0]][1]) * \
                     (sum(int(tabs[rest[1]][0][i]) for i in wb) / tabs[rest[1]][1])
                idx = np.array([(a, b) for b in wb for a in wa], dtype=np.int32)
                G, _, _ = orc.gradient(X, dims, fs, n, st, 6, idx, np.full(len(idx), pS))
                E += pS * G
                tot += pS
        assert abs(tot - 1.0) < 1e-14
        np.testing.assert_allclose(E, defs.full_gradient(X, dims, fs, n), rtol=1e-12, atol=1e-14)


def test_gradient_zero_at_exact_noiseless_factors(orc):
    """X = [[A]] -> every sampled G vanishes at A."""
    import synth

    dims = (6, 5, 4)
    fs = rand_factors(dims, 3, seed=7)
    X = synth.cp_tensor(fs)
    for strategy in S:
        st = orc.STRATEGIES[strategy]
        tabs = tables_for(orc, strategy, fs)
        for n in range(3):
            idx, w, pj = orc.sample(dims, n, st, 8, tabs, seed=1, it=n)
            G, Gam, M = orc.gradient(X, dims, fs, n, st, 8, idx, pj)
            assert np.abs(G).max() <= 1e-12 * (np.abs(fs[n] @ Gam).max() + np.abs(M).max())


def test_full_gradient_zero_at_als_solution():
    """g_bar(A*) = 0 at the ALS minimiser of eq:lsq_krp."""
    dims = (4, 5, 6)
    fs = rand_factors(dims, 3, seed=10)
    X = rand_tensor(dims, seed=11)
    for n in range(3):
        f2 = [A.copy() for A in fs]
        f2[n] = defs.als_solution(X, dims, fs, n)
        assert np.abs(defs.full_gradient(X, dims, f2, n)).max() < 1e-12


def test_single_window_block_gradient_is_full_gradient(orc):
    """one window per mode -> eq:gradient2 is g_bar deterministically."""
    dims = (4, 3, 5)
    fs = rand_factors(dims, 2, seed=13)
    X = rand_tensor(dims, seed=14)
    tabs = tables_for(orc, "block_euclidean", fs)
    idx, w, pj = orc.sample(dims, 0, orc.BLOCK_EUCLIDEAN, 15, tabs, seed=0, it=0, window=[3, 5])
    G, _, _ = orc.gradient(X, dims, fs, 0, orc.BLOCK_EUCLIDEAN, 15, idx, pj)
    np.testing.assert_allclose(G, defs.full_gradient(X, dims, fs, 0), rtol=1e-12, atol=1e-14)


def test_monte_carlo_unbiasedness(orc):
    """mean of many B=4 draws within 2% of g_bar (leverage, mode 0)."""
    dims = (4, 5, 6)
    fs = rand_factors(dims, 2, seed=15)
    X = rand_tensor(dims, seed=16)
    tabs = tables_for(orc, "leverage", fs)
    acc = np.zeros((4, 2))
    K = 20000
    for it in range(K):
        idx, w, pj = orc.sample(dims, 0, orc.LEVERAGE, 4, tabs, seed=2, it=it)
        G, _, _ = orc.gradient(X, dims, fs, 0, orc.LEVERAGE, 4, idx, pj)
        acc += G
    g = defs.full_gradient(X, dims, fs, 0)
    assert np.linalg.norm(acc / K - g) <= 0.02 * np.linalg.norm(g)


# ---------------------------------------------------------------------------------------- updates
def test_fixed_update_closed_forms(orc):
    """eq:proposed; A = I, G = I, alpha = .5 -> .5 I."""
    np.testing.assert_array_equal(orc.update_fixed(np.eye(3), np.eye(3), 0.5), 0.5 * np.eye(3))
    A = np.random.default_rng(0).standard_normal((4, 3))
    np.testing.assert_array_equal(orc.update_fixed(A, np.ones((4, 3)), 0.0), A)
    np.testing.assert_array_equal(orc.update_fixed(A, np.zeros((4, 3)), 0.7), A)


def test_adaptive_update_closed_forms(orc):
    """eq:etaada/eq:Aada: with b = eps = 0 the first step is A - eta sign(G);
    S is the running sum of G^2 and monotone; zero-G entries untouched."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((5, 3))
    G = rng.standard_normal((5, 3)); G[0, 0] = 0.0
    A1, S1 = orc.update_adaptive(A, np.zeros((5, 3)), G, 0.3)
    np.testing.assert_allclose(A1, A - 0.3 * np.sign(G), rtol=1e-15, atol=1e-15)
    np.testing.assert_array_equal(S1, G * G)
    G2 = rng.standard_normal((5, 3))
    _, S2 = orc.update_adaptive(A1, S1, G2, 0.3, b=0.5, eps=0.1)
    assert np.all(S2 >= S1)
    # b, eps > 0, a value worked by hand: A = 1, S = 1.5, G = 0.5, eta = 0.4, b = 0.5, eps = 0.25:
    # S <- 1.5 + 0.25 = 1.75; (b + S)^(1/2 + eps) = 2.25^0.75 = (1.5^2)^0.75 = 1.5^1.5 = 1.8371173070873836;
    # A <- 1 - 0.4 * 0.5 / 1.8371173070873836 = 1 - 0.10886621079036349 = 0.8911337892096365
    A4, S4 = orc.update_adaptive(np.ones((1, 1)), np.full((1, 1), 1.5), np.full((1, 1), 0.5), 0.4, b=0.5, eps=0.25)
    assert S4[0, 0] == 1.75
    assert abs(A4[0, 0] - 0.8911337892096365) <= 4e-16
    # scalar case: A=1, G=2, eta=1, b=eps=0: S=4, A <- 1 - 2/2 = 0
    A3, S3 = orc.update_adaptive(np.ones((1, 1)), np.zeros((1, 1)), 2 * np.ones((1, 1)), 1.0)
    assert A3[0, 0] == 0.0 and S3[0, 0] == 4.0


# ---------------------------------------------------------------------------------------- fit
def test_fit_closed_forms(orc):
    """fit = 1 - ||X - [[A]]||/||X|| (reading R14): X = [[A]] -> 1; zero model -> 0;
    SPEC.md:89 ones vs 0.5 ones -> relative error 0.5."""
    import synth

    dims = (3, 4, 5)
    fs = rand_factors(dims, 2, seed=3)
    X = synth.cp_tensor(fs)
    assert abs(orc.fit(X, fs) - 1.0) < 1e-14
    assert orc.fit(X, [np.zeros_like(A) for A in fs]) == 0.0
    half = [np.full((2, 1), 0.5), np.ones((2, 1)), np.ones((2, 1))]
    assert abs(orc.fit(np.ones(8), half) - 0.5) < 1e-15
    with pytest.raises(orc.OracleError):
        orc.fit(np.zeros(8), half)


def test_fit_matches_objective_definition(orc):
    dims = (3, 4, 5)
    fs = rand_factors(dims, 2, seed=17)
    X = rand_tensor(dims, seed=18)
    f = defs.objective(X, dims, fs)
    assert abs(orc.fit(X, fs) - (1 - math.sqrt(2 * f) / np.linalg.norm(X))) < 1e-13


# ---------------------------------------------------------------------------------------- end to end
def test_random_mode_uniform(orc):
    """Pr(xi = n) = 1/N: chi^2 on 30k draws."""
    N = 3
    c = np.bincount([orc.random_mode(4, r, N) for r in range(30000)], minlength=N)
    assert scipy.stats.chi2.sf(float(((c - 10000) ** 2 / 10000).sum()), N - 1) > 1e-4


@pytest.mark.parametrize("strategy", S)
def test_recovers_noiseless_exact_rank(orc, strategy):
    """Noiseless exact-rank 20^3, R = 3 (row scales exp(N(0, .5))): AdawsCPD (Alg. 7) reaches
    fit >= 0.99 (SURVEY §8c.4 end-to-end; Theorem 5.5 consequence)."""
    import synth

    cfg = synth.small((20, 20, 20), 3, batch=36, rule="adaptive", row_sigma=0.5, noise=0.0, seed=0)
    X = synth.tensor(cfg)
    A0 = synth.init_factors(cfg, X)
    fs, _, _ = orc.run(X, A0, orc.STRATEGIES[strategy], orc.STEP_ADAPTIVE, 36, 3 * 3000, window=[6, 6],
                       eta=0.3, seed=0)
    assert orc.fit(X, fs) >= 0.99


# ---------------------------------------------------------------------------------------- test helpers
@pytest.mark.parametrize("strategy", ROWWISE)
def test_gradient_from_fibers_matches_oracle(orc, strategy):
    """The full-size GPU test's reference (gpu_helpers.oracle_gradient_from_fibers over fibers read
    by gpu_helpers.gather_fibers_torch from the flat first-index-fastest tensor) equals
    oracle.tensor_samp / oracle.gradient on a small problem with a ragged mode."""
    torch = pytest.importorskip("torch")
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from gpu_helpers import gather_fibers_torch, oracle_gradient_from_fibers

    dims, R, B = (7, 5, 6), 3, 40
    fs = rand_factors(dims, R, seed=4)
    X = rand_tensor(dims, seed=5)
    tabs = tables_for(orc, strategy, fs)
    for n in range(3):
        idx, w, pj = orc.sample(dims, n, orc.STRATEGIES[strategy], B, tabs, 9, 2 + n)
        XF = gather_fibers_torch(torch.from_numpy(X), dims, n, idx)
        assert np.array_equal(XF, orc.tensor_samp(X, dims, n, idx).T)
        G, Gam, M = oracle_gradient_from_fibers(XF, dims, fs, n, strategy, B, idx, pj)
        G_o, Gam_o, M_o = orc.gradient(X, dims, fs, n, orc.STRATEGIES[strategy], B, idx, pj)
        for a, b in ((G, G_o), (Gam, Gam_o), (M, M_o)):
            assert np.allclose(a, b, rtol=1e-12, atol=1e-12 * np.abs(b).max())


# ---------------------------------------------------------------------------------------- sampled ALS step
def test_sym_pinv_closed_forms(orc):
    """Gamma^+ by the natural-order sweep: the inverse of an SPD matrix; on a rank-deficient Gram the
    Moore-Penrose conditions on the swept set (G W G = G, W G W = W) and the rank; zero -> zero."""
    rng = np.random.default_rng(21)
    Z = rng.standard_normal((40, 6))
    G = Z.T @ Z
    W, rk = orc.sym_pinv(G)
    assert rk == 6
    np.testing.assert_allclose(W, np.linalg.inv(G), rtol=1e-10, atol=1e-12 * np.abs(np.linalg.inv(G)).max())
    Z[:, 4] = 2.0 * Z[:, 1] - Z[:, 0]  # exactly dependent column (in exact arithmetic)
    G = Z.T @ Z
    W, rk = orc.sym_pinv(G)
    assert rk == 5
    np.testing.assert_allclose(G @ W @ G, G, rtol=0, atol=1e-9 * np.abs(G).max())
    np.testing.assert_allclose(W @ G @ W, W, rtol=0, atol=1e-9 * np.abs(W).max())
    W0, rk0 = orc.sym_pinv(np.zeros((3, 3)))
    assert rk0 == 0 and not W0.any()


@pytest.mark.parametrize("n", [0, 1, 2])
def test_als_step_single_window_is_exact_als(orc, n):
    """one window per mode = every fiber once: the sampled normal equations are the exact ones, so
    A = M Gamma^+ equals the ALS minimiser of eq:lsq_krp computed by lstsq."""
    dims = (4, 3, 5)
    fs = rand_factors(dims, 2, seed=31)
    X = rand_tensor(dims, seed=32)
    tabs = tables_for(orc, "block_euclidean", fs)
    win = [d for k, d in enumerate(dims) if k != n]
    B = int(np.prod(win))
    idx, w, pj = orc.sample(dims, n, orc.BLOCK_EUCLIDEAN, B, tabs, seed=0, it=0, window=win)
    _, Gam, M = orc.gradient(X, dims, fs, n, orc.BLOCK_EUCLIDEAN, B, idx, pj)
    np.testing.assert_allclose(orc.update_als(M, Gam), defs.als_solution(X, dims, fs, n), rtol=1e-10, atol=1e-12)


def test_run_wires_the_als_rule(orc):
    """oracle.run with STEP_ALS applies sample -> eq:gradient1 -> A = M Gamma^+ -> table rebuild."""
    dims = (6, 5, 4)
    fs = rand_factors(dims, 3, seed=41)
    X = rand_tensor(dims, seed=42)
    out, _, _ = orc.run(X, fs, orc.LEVERAGE, orc.STEP_ALS, 12, 2, seed=7)
    tabs = tables_for(orc, "leverage", fs)
    f = [A.copy() for A in fs]
    for it in range(2):
        n = it % 3
        idx, w, pj = orc.sample(dims, n, orc.LEVERAGE, 12, tabs, seed=7, it=it)
        _, Gam, M = orc.gradient(X, dims, f, n, orc.LEVERAGE, 12, idx, pj)
        f[n] = orc.update_als(M, Gam)
        p_, q_, T_ = orc.build_table(orc.LEVERAGE, f[n])
        tabs[n] = (q_, T_)
    for k in range(3):
        np.testing.assert_allclose(out[k], f[k], rtol=0, atol=0)


# ---------------------------------------------------------------------------------------- 8(f).1 generator
def test_spread_magnitude_generator():
    """synth.spread_magnitude (PAPER.md:683-690 with SPEC.md's stand-in rule): exact relative noise
    level, the first three columns zero except `spread` rows of +-magnitude, noiseless = [[A]]."""
    import synth

    X, X0, fs = synth.spread_magnitude(30, 12, 6, 5, 24.0, 0.05, seed=3)
    assert abs(np.linalg.norm(X - X0) / np.linalg.norm(X0) - 0.05) < 1e-12
    for A in fs:
        for c in range(3):
            nz = np.flatnonzero(A[:, c])
            assert len(nz) == 5 and np.all(np.abs(A[nz, c]) == 24.0)
    Xc, X0c, fc = synth.spread_magnitude(8, 7, 4, 0, 1.0, 0.0, seed=1)
    assert np.array_equal(Xc, X0c) and all(not A[:, :3].any() for A in fc)
    np.testing.assert_allclose(X0c, synth.cp_tensor(fc), rtol=0, atol=0)
    with pytest.raises(ValueError):
        synth.spread_magnitude(5, 4, 3, 6, 1.0)


def test_run_f32_entry_reads_the_same_tensor(orc):
    """orc_run_f32 (fp32-stored tensor, element converted to fp64 on read; the bench's C4 baseline)
    equals orc_run on the fp64 copy of the same tensor bit for bit (the conversion is exact)."""
    import synth

    cfg = synth.small((9, 8, 7), 3, dtype="f32", batch=20, rule="adaptive", seed=5, eta=0.05)
    X = synth.tensor(cfg)
    assert X.dtype == np.float32
    A0 = synth.init_factors(cfg, X)
    for st, rule in ((orc.LEVERAGE, orc.STEP_ADAPTIVE), (orc.BLOCK_EUCLIDEAN, orc.STEP_FIXED)):
        f32, S32, m32 = orc.run(X, A0, st, rule, cfg.batch, 7, eta=0.05, alpha=0.01, seed=3)
        f64, S64, m64 = orc.run(X.astype(np.float64), A0, st, rule, cfg.batch, 7, eta=0.05, alpha=0.01, seed=3)
        for a, b in zip(f32 + S32, f64 + S64):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(m32, m64)


def test_run_split_into_calls_continues_the_sweep(orc):
    """orc_run_from: 7 single-iteration calls (first mode r mod N, accumulators carried, counter r0 = r)
    equal one 7-iteration cyclic run bit for bit (the bench's bounded baseline samples run this way)."""
    import synth

    cfg = synth.small((8, 7, 6), 3, dtype="f64", batch=16, rule="adaptive", seed=2, eta=0.05)
    X = synth.tensor(cfg)
    A0 = synth.init_factors(cfg, X)
    ref, Sref, mref = orc.run(X, A0, orc.EUCLIDEAN, orc.STEP_ADAPTIVE, cfg.batch, 7, eta=0.05, seed=9)
    fs, S = A0, None
    modes = []
    for r in range(7):
        fs, S, m = orc.run(X, fs, orc.EUCLIDEAN, orc.STEP_ADAPTIVE, cfg.batch, 1, eta=0.05, seed=9, r0=r, S=S,
                           first_mode=r % 3)
        modes.append(int(m[0]))
    assert modes == list(mref)
    for a, b in zip(fs + S, ref + Sref):
        np.testing.assert_array_equal(a, b)
