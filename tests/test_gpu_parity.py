"""GPU (sm_100a) vs CPU-oracle parity, through the C ABI (libcpsgd.so via the ctypes binding).

Bars: sampled indices and weights bit-exact; integer tables equal except
entries within rounding distance of a quantisation boundary; floating point within 1e-10 (fp64)
or 1e-4 (fp32) relative, measured as ||G_gpu - G_orc|| / (||A Gamma|| + ||M||), ||dA|| / ||A||,
|d fit|.  All inputs are seeded synth data; every oracle input comes from synth.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import (S, TOL, gather_fibers_torch, handle, make_problem, near_boundary, oracle_gradient_from_fibers,
                         oracle_step, oracle_tables, rel_err, to_dev)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()


# ------------------------------------------------------------------------------------------ Philox
def test_device_philox_matches_curand_and_oracle(tmp_path):
    """device Philox == cuRAND curand_Philox4x32_10 (library routine) == oracle, 1M counters."""
    import ctypes as C

    here = os.path.dirname(os.path.abspath(__file__))
    so = str(tmp_path / "philox_check.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, os.path.join(here, "native", "philox_check.cu")])
    L = C.CDLL(so)
    n = 1 << 20
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2 ** 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    dev = torch.device("cuda:0")
    c = torch.from_numpy(ctr.view(np.int32)).to(dev)
    k = torch.from_numpy(key.view(np.int32)).to(dev)
    ours = torch.zeros((n, 4), dtype=torch.int32, device=dev)
    theirs = torch.zeros((n, 4), dtype=torch.int32, device=dev)
    assert L.philox_check(C.c_void_p(c.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(ours.data_ptr()),
                          C.c_void_p(theirs.data_ptr()), n) == 0
    o = ours.cpu().numpy().view(np.uint32)
    t = theirs.cpu().numpy().view(np.uint32)
    assert np.array_equal(o, t)
    for i in rng.integers(0, n, size=200):
        assert oracle.philox(ctr[i], key[i]).tolist() == o[i].tolist()


# ------------------------------------------------------------------------------------------ tables
@pytest.mark.parametrize("strategy", ["leverage", "euclidean", "block_leverage", "block_euclidean"])
@pytest.mark.parametrize("cfgname", ["C1", "C2", "C3"])
def test_tables_match_oracle(strategy, cfgname):
    """a1: GPU p vs oracle p <= 1e-11 relative; integer q identical except near-boundary entries."""
    cfg = synth.CONFIGS[cfgname]
    A_true = synth.true_factors(cfg)
    A = [np.ascontiguousarray(a.astype(np.float64 if cfg.dtype == "f64" else np.float32)) for a in A_true]
    dev = torch.device("cuda:0")
    Ad = [torch.from_numpy(a).to(dev) for a in A]
    Xd = torch.zeros(int(np.prod(cfg.dims)), dtype=Ad[0].dtype, device=dev)  # tables read only the factors
    h = handle(cfg, Xd, Ad, strategy, mode_major=False)
    tabs = oracle_tables(strategy, A)
    for k in range(cfg.order):
        q, T, p = h.get_table(k)
        po, qo, To = tabs[k]
        assert np.all(np.abs(p - po) <= 1e-11 * po + 1e-300), np.max(np.abs(p - po) / po)
        diff = q != qo
        flip_ok = near_boundary(po, 1e-3)
        assert np.all(~diff | flip_ok)
        assert np.all(np.abs(q.astype(np.int64) - qo.astype(np.int64)) <= 1)
        assert T == int(q.sum())
    h.close()


# ------------------------------------------------------------------------------------------ sampler
@pytest.mark.parametrize("strategy", S)
@pytest.mark.parametrize("dims,R,B", [((60, 60, 60), 5, 64), ((33, 17, 41), 4, 100), ((11, 9, 13, 7), 3, 256)])
def test_sample_bit_exact(strategy, dims, R, B):
    """a2/a3: idx and omega identical to the oracle's for every mode and several iterations."""
    cfg = synth.small(dims, R, batch=B, rule="fixed", row_sigma=1.0, seed=5)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, strategy, seed=123)
    tabs = oracle_tables(strategy, A0)
    tq = [(t[1], t[2]) for t in tabs]
    for k in range(len(dims)):
        qg, Tg, _ = h.get_table(k)
        assert np.array_equal(qg, tabs[k][1]) and Tg == tabs[k][2], "table flip (rare); pick another seed"
    for n in range(len(dims)):
        for it in (0, 1, 7, 2 ** 33 + 5):
            idx_g, w_g = h.sample(n, it)
            idx_o, w_o, _ = oracle.sample(dims, n, oracle.STRATEGIES[strategy], B, tq, 123, it)
            assert np.array_equal(idx_g.cpu().numpy(), idx_o)
            assert np.array_equal(w_g.cpu().numpy(), w_o)
    h.close()


# ------------------------------------------------------------------------------------------ one step
STEP_CASES = [
    # (dims, R, B, dtype, rule)
    ((60, 60, 60), 5, 64, "f64", "fixed"),           # C1 shape
    ((130, 70, 45), 20, 512, "f32", "adaptive"),     # C2-like, ragged I-tiles (130 = 128 + 2)
    ((20, 18, 16, 14), 10, 1024, "f32", "adaptive"),  # C3-like 4-way
    ((9, 1, 7), 3, 5, "f64", "fixed"),               # a unit mode, tiny batch
    ((40, 30, 20), 1, 1, "f64", "adaptive"),         # R = 1, B = 1
    ((50, 40, 30), 64, 300, "f32", "fixed"),         # R = 64 (max)
]


PATHS = {"fused": dict(fused=True, mode_major=True),            # persistent single-cluster kernel
         "fused_cu8": dict(fused=True, mode_major=True, fused_cluster=8),  # same on 8-CTA clusters
         "split_mm": dict(fused=False, mode_major=True),        # gather+update kernel, then table/sample kernel
         "split_native": dict(fused=False, mode_major=False),   # same, strided fibers in the native layout
         "split_ffma": dict(fused=False, tc=False, mode_major=True),  # wide path, FFMA mainloop (no tcgen05)
         "legacy_mm": dict(fused=False, wide=False, mode_major=True)}  # gather partials + update/table/sample


@pytest.mark.parametrize("strategy", S)
@pytest.mark.parametrize("case", STEP_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_R{c[1]}_B{c[2]}_{c[3]}")
@pytest.mark.parametrize("path", list(PATHS))
def test_one_step_per_mode(strategy, case, path):
    """a4-a8: from the same seeded state, one GPU step of mode n at iteration r equals one oracle
    step: G within tol of (||A Gamma|| + ||M||), updated A within tol of ||A||."""
    dims, R, B, dt, rule = case
    cfg = synth.small(dims, R, dtype=dt, batch=B, rule=rule, row_sigma=1.0, noise=1e-2, seed=11, alpha=0.01,
                      eta=0.05)
    bpar = 1e-2  # b > 0 keeps the first AdaGrad step smooth in G (b = 0 gives eta*sign(G))
    X, A0 = make_problem(cfg)
    tol = TOL[dt]
    for n in range(len(dims)):
        Xd, Ad = to_dev(X, A0)
        h = handle(cfg, Xd, Ad, strategy, seed=77, b=bpar, **PATHS[path])
        it = 3 + n
        h.iter = it
        idx_o, w_o, G_o, Gam_o, M_o, tabs = oracle_step(X, dims, A0, n, strategy, B, 77, it)
        h.step(n, cfg.alpha)
        G_g, m, Gam_g = h.get_grad()
        assert m == n and h.iter == it + 1
        A64 = np.asarray(A0[n], np.float64)
        scale = np.linalg.norm(A64 @ Gam_o) + np.linalg.norm(M_o)
        assert rel_err(G_g, G_o, scale) <= tol
        assert rel_err(Gam_g, Gam_o, np.linalg.norm(Gam_o)) <= tol
        if rule == "fixed":
            A_o = oracle.update_fixed(A64, G_o, cfg.alpha)
        else:
            A_o, S_o = oracle.update_adaptive(A64, np.zeros_like(A64), G_o, cfg.eta, b=bpar)
            S_g = h.get_accum(n)
            assert rel_err(S_g, S_o, np.linalg.norm(S_o)) <= 2 * tol
        A_g = Ad[n].cpu().numpy()
        assert rel_err(A_g, A_o, np.linalg.norm(A_o)) <= tol
        for k in range(len(dims)):
            if k != n:
                assert np.array_equal(Ad[k].cpu().numpy(), A0[k])
        h.close()


# ------------------------------------------------------------------------------------------ sampled ALS step (8f.3)
ALS_CASES = [((60, 60, 60), 5, 64, "f64"), ((40, 30, 20), 12, 300, "f64"), ((130, 70, 45), 20, 512, "f32")]


@pytest.mark.parametrize("strategy", ["uniform", "leverage", "euclidean", "block_leverage"])
@pytest.mark.parametrize("case", ALS_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_R{c[1]}_B{c[2]}_{c[3]}")
@pytest.mark.parametrize("path", ["fused", "split_mm", "split_ffma"])
def test_als_step_per_mode(strategy, case, path):
    """rule=als: one GPU step of mode n equals A = M Gamma^+ of the oracle from the same state; the
    tolerance is the dtype's times the condition number of Gamma, the
    factor by which a solve can amplify the input perturbation."""
    dims, R, B, dt = case
    cfg = synth.small(dims, R, dtype=dt, batch=B, rule="fixed", row_sigma=1.0, noise=1e-2, seed=13)
    X, A0 = make_problem(cfg)
    for n in range(len(dims)):
        Xd, Ad = to_dev(X, A0)
        h = handle(cfg, Xd, Ad, strategy, seed=55, rule="als", **PATHS[path])
        it = 2 + n
        h.iter = it
        idx_o, w_o, G_o, Gam_o, M_o, tabs = oracle_step(X, dims, A0, n, strategy, B, 55, it)
        h.step(n)
        A_o = oracle.update_als(M_o, Gam_o)
        kappa = np.linalg.cond(Gam_o)
        A_g = Ad[n].cpu().numpy()
        assert rel_err(A_g, A_o, np.linalg.norm(A_o)) <= TOL[dt] * max(1.0, kappa)
        for k in range(len(dims)):
            if k != n:
                assert np.array_equal(Ad[k].cpu().numpy(), A0[k])
        h.close()


@pytest.mark.parametrize("path", ["fused", "split_mm"])
def test_als_trajectory(path):
    """rule=als, C1 shape (60^3 fp64, R5, B64, leverage), 4 cyclic sweeps free-running on both
    sides: final factors within 1e-8 relative."""
    cfg = synth.small((60, 60, 60), 5, dtype="f64", batch=64, rule="fixed", row_sigma=1.0, noise=1e-2, seed=0)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=3, rule="als", **PATHS[path])
    h.sweep(4)
    h.sync()
    fs, _, _ = oracle.run(X, A0, oracle.LEVERAGE, oracle.STEP_ALS, cfg.batch, 12, seed=3)
    for k in range(3):
        assert rel_err(Ad[k].cpu().numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-8
    h.close()


def test_als_needs_fused_or_wide_path():
    from paper_2103_04081_b200 import CPError

    cfg = synth.small((20, 18, 16), 3, dtype="f64", batch=32, rule="fixed", seed=2)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    with pytest.raises(CPError, match="EINVAL"):
        handle(cfg, Xd, Ad, "leverage", rule="als", fused=False, wide=False)


# ------------------------------------------------------------------------------------------ multi-chain (8f.2)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_multi_chain_sweeps_equal_separate_runs(dt):
    """cp_sgd_sweep_multi: four chains (different samplers, seeds, rules) in one launch equal four
    separate cp_sgd_sweep calls bit for bit (the same per-cluster code on the same inputs)."""
    from paper_2103_04081_b200 import CPSGD

    cfg = synth.small((40, 30, 20), 6, dtype=dt, batch=64, rule="adaptive", eta=0.05, seed=4)
    X, A0 = make_problem(cfg)
    specs = [("leverage", 1, "adaptive"), ("euclidean", 2, "fixed"), ("uniform", 3, "adaptive"),
             ("block_leverage", 4, "als")]
    ref = []
    for s, seed, rule in specs:
        Xd, Ad = to_dev(X, A0)
        h = handle(cfg, Xd, Ad, s, seed=seed, rule=rule)
        h.sweep(3)
        h.sync()
        ref.append([a.cpu().numpy() for a in Ad])
        h.close()
    hs, Ads, Xs = [], [], []
    for s, seed, rule in specs:
        Xd, Ad = to_dev(X, A0)
        hs.append(handle(cfg, Xd, Ad, s, seed=seed, rule=rule))
        Ads.append(Ad)
        Xs.append(Xd)
    CPSGD.sweep_multi(hs, 3)
    for i, h in enumerate(hs):
        h.sync()
        assert h.iter == 9
        for k in range(3):
            assert np.array_equal(Ads[i][k].cpu().numpy(), ref[i][k])
    if dt == "f64":  # and every chain equals the oracle's own run of it (Alg. 6 / 7, sampled ALS)
        rules = {"fixed": oracle.STEP_FIXED, "adaptive": oracle.STEP_ADAPTIVE, "als": oracle.STEP_ALS}
        for i, (s, seed, rule) in enumerate(specs):
            fs, _, _ = oracle.run(X, A0, oracle.STRATEGIES[s], rules[rule], cfg.batch, 9, alpha=cfg.alpha, eta=cfg.eta,
                                  seed=seed)
            tol = 1e-8 if rule == "als" else 1e-10
            for k in range(3):
                assert rel_err(Ads[i][k].cpu().numpy(), fs[k], np.linalg.norm(fs[k])) <= tol, (s, rule, k)
    # a handle of another geometry is refused
    cfg2 = synth.small((40, 30, 21), 6, dtype=dt, batch=64, rule="adaptive", eta=0.05, seed=4)
    X2, A2 = make_problem(cfg2)
    Xd2, Ad2 = to_dev(X2, A2)
    h2 = handle(cfg2, Xd2, Ad2, "leverage", seed=9)
    from paper_2103_04081_b200 import CPError

    with pytest.raises(CPError, match="EINVAL"):
        CPSGD.sweep_multi([hs[0], h2], 1)
    for h in hs + [h2]:
        h.close()


# ------------------------------------------------------------------------------------------ trajectories
@pytest.mark.parametrize("strategy", S)
@pytest.mark.parametrize("path", ["fused", "split_mm"])
def test_c1_trajectory_50_sweeps(strategy, path):
    """C1 (60^3 fp64, R5, B64, fixed alpha, 50 cyclic sweeps) free-running on both sides: final
    factors within 1e-9 relative (one persistent launch, or graph-replayed split sweeps)."""
    cfg = synth.CONFIGS["C1"]
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, strategy, seed=0, **PATHS[path])
    h.sweep(50)
    h.sync()
    fs, _, _ = oracle.run(X, A0, oracle.STRATEGIES[strategy], oracle.STEP_FIXED, cfg.batch, 50 * 3,
                          alpha=cfg.alpha, seed=0)
    for k in range(3):
        assert rel_err(Ad[k].cpu().numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-9
    assert abs(h.fit() - oracle.fit(X, fs)) <= 1e-9
    assert h.iter == 150
    h.close()


@pytest.mark.parametrize("strategy", ["leverage", "block_euclidean"])
@pytest.mark.parametrize("path", ["fused", "split_mm"])
def test_random_order_and_adaptive_trajectory(strategy, path):
    """random mode order, adaptive rule, fp64: 40 iterations equal the oracle's."""
    cfg = synth.small((24, 20, 16), 4, dtype="f64", batch=48, rule="adaptive", eta=0.05, seed=3, row_sigma=0.8)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, strategy, seed=9, **PATHS[path])
    h.sweep(40 // 3 + 1, order="random")
    iters = 3 * (40 // 3 + 1)
    fs, Ss, modes = oracle.run(X, A0, oracle.STRATEGIES[strategy], oracle.STEP_ADAPTIVE, cfg.batch, iters,
                               order=oracle.ORDER_RANDOM, eta=cfg.eta, seed=9)
    for k in range(3):
        assert rel_err(Ad[k].cpu().numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-9
        assert rel_err(h.get_accum(k), Ss[k], np.linalg.norm(Ss[k]) + 1e-300) <= 1e-9
    h.close()


def test_fixed_schedule_sweep_matches_oracle():
    """per-iteration step sizes alpha_r = a0 / (1 + r)^0.6 (Robbins-Monro)."""
    cfg = synth.small((30, 25, 20), 5, dtype="f64", batch=40, rule="fixed", seed=4)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "euclidean", seed=1)
    al = 0.01 / (1.0 + np.arange(12)) ** 0.6
    h.sweep(4, alphas=al)
    fs, _, _ = oracle.run(X, A0, oracle.EUCLIDEAN, oracle.STEP_FIXED, cfg.batch, 12, alphas=al, seed=1)
    for k in range(3):
        assert rel_err(Ad[k].cpu().numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-9
    h.close()


# ------------------------------------------------------------------------------------------ fit
@pytest.mark.parametrize("cfgname", ["C1", "C3"])
def test_fit_matches_oracle(cfgname):
    cfg = synth.CONFIGS[cfgname]
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage")
    assert abs(h.fit() - oracle.fit(X, A0)) <= TOL[cfg.dtype]
    # the exact model gives fit 1 (noiseless)
    cfg0 = synth.small((17, 13, 11), 3, dtype=cfg.dtype, noise=0.0, seed=2)
    At = [a.astype(np.float64 if cfg.dtype == "f64" else np.float32) for a in synth.true_factors(cfg0)]
    X0 = synth.cp_tensor(At).astype(At[0].dtype)
    Xd0, Ad0 = to_dev(X0, At)
    h0 = handle(cfg0, Xd0, Ad0, "leverage")
    assert abs(h0.fit() - 1.0) <= TOL[cfg.dtype]
    h.close(); h0.close()


# ------------------------------------------------------------------------------------------ full size (bench config)
@pytest.mark.parametrize("path", ["fused", "split_mm"])
def test_c2_full_size_step_and_fit(path):
    """C2 at full size (400^3 fp32, R20, B512, adaptive) in the launch configuration bench.py
    times (fused), and the split path: one step per mode vs the oracle, and fit."""
    cfg = synth.CONFIGS["C2"]
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=0)
    assert abs(h.fit() - oracle.fit(X, A0)) <= 1e-4
    h.close()
    del Xd
    for n in range(3):
        Xd, Ad = to_dev(X, A0)
        h = handle(cfg, Xd, Ad, "leverage", seed=0, **PATHS[path])
        h.iter = n
        idx_o, w_o, G_o, Gam_o, M_o, tabs = oracle_step(X, cfg.dims, A0, n, "leverage", cfg.batch, 0, n)
        idx_g, w_g = h.sample(n, n)
        assert np.array_equal(idx_g.cpu().numpy(), idx_o) and np.array_equal(w_g.cpu().numpy(), w_o)
        h.step(n)
        G_g, _, _ = h.get_grad()
        scale = np.linalg.norm(np.asarray(A0[n], np.float64) @ Gam_o) + np.linalg.norm(M_o)
        assert rel_err(G_g, G_o, scale) <= 1e-4
        h.close()
        del Xd


def test_c4_full_size_tcgen05_step():
    """C4 at full size (2000^3 fp32 = 32 GB, R50, B4096, leverage) through the wide tcgen05 path in
    the launch configuration bench.py --workload C4 times: sampled indices and weights bit-exact,
    G and Gamma within 1e-4 of the oracle from the same seeded input (the oracle reads the sampled
    fibers of the seeded tensor; its SKR rows, weights and scale are its own)."""
    cfg = synth.CONFIGS["C4"]
    dev = torch.device("cuda:0")
    Xd, _, xn = synth.tensor_torch(cfg, device=dev)
    Ad0 = synth.init_factors_torch(cfg, xn, device=dev)
    A0 = [a.cpu().numpy() for a in Ad0]
    tabs = oracle_tables("leverage", A0)
    tq = [(t[1], t[2]) for t in tabs]
    for n in range(3):
        Ad = [a.clone() for a in Ad0]
        h = handle(cfg, Xd, Ad, "leverage", seed=0, fused=False, mode_major=True)
        h.iter = n
        idx_o, w_o, pj = oracle.sample(cfg.dims, n, oracle.STRATEGIES["leverage"], cfg.batch, tq, 0, n)
        idx_g, w_g = h.sample(n, n)
        assert np.array_equal(idx_g.cpu().numpy(), idx_o) and np.array_equal(w_g.cpu().numpy(), w_o)
        h.step(n)
        G_g, m, Gam_g = h.get_grad()
        assert m == n
        XF = gather_fibers_torch(Xd, cfg.dims, n, idx_o)
        G_o, Gam_o, M_o = oracle_gradient_from_fibers(XF, cfg.dims, A0, n, "leverage", cfg.batch, idx_o, pj)
        scale = np.linalg.norm(np.asarray(A0[n], np.float64) @ Gam_o) + np.linalg.norm(M_o)
        assert rel_err(G_g, G_o, scale) <= 1e-4
        assert rel_err(Gam_g, Gam_o, np.linalg.norm(Gam_o)) <= 1e-4
        h.close()
        del Ad
        torch.cuda.empty_cache()


# ------------------------------------------------------------------------------------------ e2e host path
@pytest.mark.parametrize("fused", [True, False])
def test_steps_host_takes_over_changed_factors(fused):
    """cp_sgd_steps_host with host factors that differ from the device copy (one mode changed, then
    all): the changed factors replace the device ones and their tables are rebuilt before the steps."""
    cfg = synth.small((30, 20, 10), 4, dtype="f64", batch=32, rule="fixed", seed=8)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=2, fused=fused)
    rng = np.random.default_rng(5)
    A1 = [a.copy() for a in A0]
    A1[1] = A1[1] * np.exp(0.3 * rng.standard_normal(A1[1].shape))  # one mode changed
    host = [torch.from_numpy(a.copy()).pin_memory() for a in A1]
    h.steps_host(0, 3, host, 0.01)
    fs, _, _ = oracle.run(X, A1, oracle.LEVERAGE, oracle.STEP_FIXED, cfg.batch, 3, alpha=0.01, seed=2)
    for k in range(3):
        assert rel_err(host[k].numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-10
    A2 = [a * (1.0 + 0.1 * rng.standard_normal(a.shape)) for a in fs]  # every mode changed
    host = [torch.from_numpy(a.copy()).pin_memory() for a in A2]
    h.steps_host(0, 3, host, 0.01)
    fs2, _, _ = oracle.run(X, A2, oracle.LEVERAGE, oracle.STEP_FIXED, cfg.batch, 3, alpha=0.01, seed=2, r0=3)
    for k in range(3):
        assert rel_err(host[k].numpy(), fs2[k], np.linalg.norm(fs2[k])) <= 1e-10
    h.close()


def test_steps_host_equals_device_path():
    cfg = synth.small((30, 20, 10), 4, dtype="f64", batch=32, rule="fixed", seed=8)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=2)
    host = [torch.from_numpy(a.copy()).pin_memory() for a in A0]
    h.steps_host(0, 6, host, 0.01)
    fs, _, _ = oracle.run(X, A0, oracle.LEVERAGE, oracle.STEP_FIXED, cfg.batch, 6, alpha=0.01, seed=2)
    for k in range(3):
        assert rel_err(host[k].numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-10
    h.close()


# ------------------------------------------------------------------------------------------ errors
def test_error_paths():
    from paper_2103_04081_b200 import CPError

    cfg = synth.small((8, 7, 6), 2, dtype="f64", batch=4, seed=1)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    with pytest.raises(CPError, match="EINVAL"):
        handle(cfg, Xd, Ad, "leverage", rule="adaptive", eta=0.0)
    Z = [torch.zeros_like(a) for a in Ad]
    with pytest.raises(CPError, match="EDEGENERATE"):
        handle(cfg, Xd, Z, "euclidean")
    Nn = [a.clone() for a in Ad]
    Nn[1][0, 0] = float("nan")
    with pytest.raises(CPError, match="ENONFINITE"):
        handle(cfg, Xd, Nn, "leverage")
    h = handle(cfg, Xd, Ad, "leverage")
    with pytest.raises(CPError, match="ERANGE"):
        h.step(3)
    # a diverging step poisons the next table rebuild -> reported at the next sync
    h.step(0, float("inf"))
    with pytest.raises(CPError, match="ENONFINITE|EDEGENERATE"):
        h.sync()
    h.close()
