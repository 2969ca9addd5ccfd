"""Parity of the batches the BENCHED launches actually consume, at full size (VERDICT r01 "parity"):
the debug trace (cp_sgd_trace) records, for every SGD iteration a persistent kernel runs, the batch it
drew and the factor / accumulator / table it left; the oracle replays each iteration from the traced
state (teacher forcing):

* C2 (400^3 fp32, R20, B512, adaptive, leverage) on the fused single-cluster kernel -- bench.py
  --workload C2 -- over a 20-sweep run (60 iterations in one launch);
* C4 (2000^3 fp32 = 32 GB, R50, B4096, adaptive, leverage) on the persistent cooperative kernel --
  bench.py's default workload -- over 2 sweeps;
* C3 (100^4 fp32, R10, B1024, adaptive) one step per mode at full size on its benched (fused) path.

Bars: indices and weights bit-exact against oracle.sample on the GPU's integer tables; tables equal
to the oracle's table of the traced factor except entries at a rounding boundary; updates within
the fp32 tolerance (Frobenius and per-row), b = 0 sign-sensitive entries masked (gpu_helpers.trace_check).
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import (TOL, gather_fibers_torch, handle, make_problem, oracle_gradient_from_fibers, oracle_step,
                         oracle_tables, rel_err, row_rel_err, to_dev, trace_check)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()


def test_c2_fused_20_sweeps_traced():
    cfg = synth.CONFIGS["C2"]
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=0)
    assert h.path == "fused"
    h.trace_start(60)
    h.sweep(20)
    recs = h.trace_read()
    assert len(recs) == 60 and [r["n"] for r in recs] == [0, 1, 2] * 20
    assert [r["r"] for r in recs] == list(range(60))
    q0 = [t[1] for t in oracle_tables("leverage", A0)]
    X64 = X.astype(np.float64)
    masked = trace_check(X64, cfg.dims, A0, recs, "leverage", cfg.batch, 0, "adaptive", cfg, q0)
    print("masked sign-sensitive entries:", masked)
    for k in range(3):
        last = max(i for i, r in enumerate(recs) if r["n"] == k)
        assert np.array_equal(Ad[k].cpu().numpy(), recs[last]["A"])
    h.close()


def test_c4_persistent_traced():
    cfg = synth.CONFIGS["C4"]
    dev = torch.device("cuda:0")
    Xd, _, xn = synth.tensor_torch(cfg, device=dev)
    Ad = synth.init_factors_torch(cfg, xn, device=dev)
    A0 = [a.cpu().numpy() for a in Ad]
    h = handle(cfg, Xd, Ad, "leverage", seed=0, fused=False, mode_major=True)
    assert h.path == "persistent"
    h.trace_start(6)
    h.sweep(2)
    recs = h.trace_read()
    assert [r["n"] for r in recs] == [0, 1, 2, 0, 1, 2]

    def grad(A, n, idx, pj):
        XF = gather_fibers_torch(Xd, cfg.dims, n, idx)
        return oracle_gradient_from_fibers(XF, cfg.dims, A, n, "leverage", cfg.batch, idx, pj)

    q0 = [t[1] for t in oracle_tables("leverage", A0)]
    trace_check(None, cfg.dims, A0, recs, "leverage", cfg.batch, 0, "adaptive", cfg, q0, grad=grad)
    h.close()
    del Xd, Ad
    torch.cuda.empty_cache()


def test_c3_full_size_one_step_per_mode():
    """C3 (4-way 100^4 fp32, R10, B1024, adaptive, b = 0 as benched): G, Gamma, A, S after one step of
    each mode from the seeded state, on the benched (fused) path."""
    cfg = synth.CONFIGS["C3"]
    X, A0 = make_problem(cfg)
    X64 = X.astype(np.float64)
    for n in range(4):
        Xd, Ad = to_dev(X, A0)
        h = handle(cfg, Xd, Ad, "leverage", seed=4)
        assert h.path == "fused"
        h.iter = 10 + n
        idx_o, w_o, G_o, Gam_o, M_o, _ = oracle_step(X64, cfg.dims, A0, n, "leverage", cfg.batch, 4, 10 + n)
        h.trace_start(1)
        h.step(n)
        rec = h.trace_read()[0]
        assert np.array_equal(rec["idx"], idx_o) and np.array_equal(rec["w"], w_o)
        G_g, m, Gam_g = h.get_grad()
        A64 = np.asarray(A0[n], np.float64)
        scale = np.linalg.norm(A64 @ Gam_o) + np.linalg.norm(M_o)
        assert rel_err(G_g, G_o, scale) <= TOL["f32"]
        assert rel_err(Gam_g, Gam_o, np.linalg.norm(Gam_o)) <= TOL["f32"]
        # b = 0: the first AdaGrad step is eta sign(G): entries with |G| inside the tolerance band masked
        A_o, S_o = oracle.update_adaptive(A64, np.zeros_like(A64), G_o, cfg.eta)
        band = np.abs(G_o) <= 10 * TOL["f32"] * scale / np.sqrt(G_o.size)
        assert band.mean() < 0.01
        A_g = Ad[n].cpu().numpy().astype(np.float64)
        assert np.linalg.norm(np.where(band, 0.0, A_g - A_o)) <= TOL["f32"] * np.linalg.norm(A_o)
        assert row_rel_err(np.where(band, A_o, A_g), A_o) <= 10 * TOL["f32"]
        assert rel_err(h.get_accum(n), S_o, np.linalg.norm(S_o)) <= 2 * TOL["f32"]
        h.close()
        del Xd


def exchange_rows(buf, I, R):
    """the library's phase-0 exchange buffer of a wide-path rank ([ceil(I/128)][R][128]: its chunk sum of
    M^T by 128-row tile) as the I x R matrix"""
    t = (I + 127) // 128
    return np.asarray(buf, np.float64).reshape(t, R, 128).transpose(1, 0, 2).reshape(R, t * 128)[:, :I].T


def test_c5_slab_rank0_full_size():
    """C5 (4000^3 fp32 = 256 GB, R32, B8192, adaptive): rank 0 of the 8-way slab split run on one GPU -- its
    32 GB slab X[..., 0:500] (+ mode-major copies), an external-comm handle.  The global batch is bit-exact
    with the oracle; phase 0 of mode 0 leaves the partial M over the fibers the rank owns (i_3 in its slab);
    phases 0-1 of the last mode update the rank's rows A^(3)[0:500] from its fiber segments -- both against the
    oracle's gradient on the same sampled fibers read from the seeded slab (fp32 tolerance; b = 0 band mask)."""
    from paper_2103_04081_b200 import CPSGD
    from paper_2103_04081_b200.parallel import slab_ranges

    cfg = synth.CONFIGS["C5"]
    dims, R, B = cfg.dims, cfg.rank, cfg.batch
    lo, hi = slab_ranges(dims[-1], 8)[0]
    ldims = (dims[0], dims[1], hi - lo)
    dev = torch.device("cuda:0")
    Xd, _, xn = synth.tensor_torch(cfg, device=dev, slab=(lo, hi))
    Ad = synth.init_factors_torch(cfg, xn, device=dev)
    A0 = [a.cpu().numpy() for a in Ad]
    fs = [np.asarray(a, np.float64) for a in A0]
    h = CPSGD(Xd, dims, Ad, B, sampler="leverage", rule="adaptive", eta=cfg.eta, seed=2, world_rank=0, world_size=8,
              slab=(lo, hi), external_comm=True, fused=False)
    tabs = oracle_tables("leverage", A0)
    tq = [(t[1], t[2]) for t in tabs]
    Jn = float(dims[1] * dims[2])
    # ---- mode 0 at r = 0: the batch, then the partial M over the owned fibers ----
    idx_o, w_o, pj = oracle.sample(dims, 0, oracle.LEVERAGE, B, tq, 2, 0)
    ig, wg = h.sample(0, 0)
    assert np.array_equal(ig.cpu().numpy(), idx_o) and np.array_equal(wg.cpu().numpy(), w_o)
    h.step_phase(0, 0)
    buf = torch.empty(h.exchange_count(0), dtype=torch.float32, device=dev)
    h.exchange_copy(0, buf, False)
    M_g = exchange_rows(buf.cpu().numpy(), dims[0], R)
    own = (idx_o[:, 1] >= lo) & (idx_o[:, 1] < hi)
    li = idx_o[own].copy()
    li[:, 1] -= lo
    XF = gather_fibers_torch(Xd, ldims, 0, li)                     # (owned, I_0) from the seeded slab
    Z = oracle.skr(fs, 0, idx_o[own])
    d = 1.0 / pj[own]
    M_o = (XF.T @ (d[:, None] * Z)) / (B * Jn)
    assert 0.05 < own.mean() < 0.3                                 # the slab's share of the leverage mass
    assert rel_err(M_g, M_o, np.linalg.norm(M_o)) <= TOL["f32"]
    assert row_rel_err(M_g, M_o) <= 10 * TOL["f32"]
    h.close()
    # ---- the last mode at r = 1: every fiber's slab segment, the rank's rows of A^(3) updated ----
    h = CPSGD(Xd, dims, Ad, B, sampler="leverage", rule="adaptive", eta=cfg.eta, seed=2, world_rank=0, world_size=8,
              slab=(lo, hi), external_comm=True, fused=False)
    h.iter = 1
    idx_o, w_o, pj = oracle.sample(dims, 2, oracle.LEVERAGE, B, tq, 2, 1)
    h.step_phase(2, 0)
    h.step_phase(2, 1)
    torch.cuda.synchronize()
    XF = gather_fibers_torch(Xd, ldims, 2, idx_o)                 # (B, 500): the fibers' slab segments
    Z = oracle.skr(fs, 2, idx_o)
    d = 1.0 / pj
    scale = 1.0 / (B * float(dims[0] * dims[1]))
    C1 = Z.T @ (d[:, None] * Z)
    C2 = XF.T @ (d[:, None] * Z)
    Arows = fs[2][lo:hi]
    G_o = scale * (Arows @ C1 - C2)
    A_o, _ = oracle.update_adaptive(Arows, np.zeros_like(Arows), G_o, cfg.eta)
    sc = np.linalg.norm(scale * (Arows @ C1)) + np.linalg.norm(scale * C2)
    band = np.abs(G_o) <= 10 * TOL["f32"] * sc / np.sqrt(G_o.size)  # b = 0: eta sign(G) (gpu_helpers.trace_check)
    assert band.mean() < 0.05
    A_g = Ad[2][lo:hi].cpu().numpy().astype(np.float64)
    assert np.linalg.norm(np.where(band, 0.0, A_g - A_o)) <= TOL["f32"] * np.linalg.norm(A_o)
    assert row_rel_err(np.where(band, A_o, A_g), A_o) <= 10 * TOL["f32"]
    assert np.array_equal(Ad[2][hi:].cpu().numpy(), A0[2][hi:])   # rows of the other ranks: untouched
    h.close()
    del Xd, Ad
    torch.cuda.empty_cache()
