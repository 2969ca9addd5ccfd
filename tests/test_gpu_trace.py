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
