"""The persistent cooperative sweep kernel of the fp32 wide path (k_sweep_wide) -- the launch bench.py
times at C4 -- against the CPU oracle, through the C ABI.

* one step per mode from the same seeded state (every strategy, ragged tiles, R up to 64);
* the debug trace of several cyclic sweeps: every consumed batch bit-exact against oracle.sample fed
  with the GPU's integer tables of that moment (teacher-forced tables), every rebuilt table equal to
  the oracle's table of the traced factor except near-boundary entries, and every update within the
  fp32 tolerance of the oracle's step from the traced state (teacher forcing);
* block strategies, random mode order, per-iteration step schedules.

Bars: indices and weights bit-exact; G / A / S within 1e-4 relative
(Frobenius) and a per-row bound; tables within one unit of q only at a rounding boundary.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import (S, TOL, handle, make_problem, near_boundary, oracle_step, oracle_tables, rel_err,
                         row_rel_err, to_dev, trace_check)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()


PW_CASES = [
    # dims, R, B
    ((300, 130, 200), 50, 4096),    # C4 shape in miniature: ragged I-tiles (300 = 2*128 + 44), 9 chunks
    ((260, 140, 96), 20, 512),      # C2-like rank and batch
    ((132, 70, 45), 48, 1000),      # R = 48, ragged batch (1000 = 31 units + 8); I_2 = 45 < 2R
    ((200, 64, 33, 20), 10, 1024),  # 4-way
    ((2600, 40, 30), 16, 1024),     # I_0 > 148 x 16: CTAs with two row units (shared rows re-read, prefix loop)
    ((260, 140, 130), 64, 1024),    # R = 64 = kMaxRank (the RMAX = 64 sweep instance)
    ((200, 120, 80), 33, 768),      # R = 33: the smallest rank on the fp64 tensor-core phases (most 8x8 tiles padding)
    ((240, 160, 120), 56, 1024),    # R = 56 = RMAX: no padding column in the last 8x8 block
    ((120, 96, 84, 20), 40, 512),   # 4-way (the generic sampling code) with the tensor-core phases; I_3 < 2R
]


@pytest.mark.parametrize("strategy", S)
@pytest.mark.parametrize("case", PW_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_R{c[1]}_B{c[2]}")
@pytest.mark.parametrize("rule", ["fixed", "adaptive"])
def test_pw_one_step_per_mode(strategy, case, rule):
    dims, R, B = case
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule=rule, row_sigma=1.0, noise=1e-2, seed=21, alpha=0.01,
                      eta=0.05)
    X, A0 = make_problem(cfg)
    bpar = 1e-2
    for n in range(len(dims)):
        Xd, Ad = to_dev(X, A0)
        h = handle(cfg, Xd, Ad, strategy, seed=31, b=bpar, fused=False, mode_major=True)
        assert h.path == "persistent"
        it = 5 + n
        h.iter = it
        idx_o, w_o, G_o, Gam_o, M_o, tabs = oracle_step(X, dims, A0, n, strategy, B, 31, it)
        h.trace_start(1)
        h.step(n, cfg.alpha)
        rec = h.trace_read()[0]
        assert rec["n"] == n and rec["r"] == it
        assert np.array_equal(rec["idx"], idx_o) and np.array_equal(rec["w"], w_o)
        G_g, m, Gam_g = h.get_grad()
        assert m == n and h.iter == it + 1
        A64 = np.asarray(A0[n], np.float64)
        scale = np.linalg.norm(A64 @ Gam_o) + np.linalg.norm(M_o)
        assert rel_err(G_g, G_o, scale) <= TOL["f32"]
        assert rel_err(Gam_g, Gam_o, np.linalg.norm(Gam_o)) <= TOL["f32"]
        if rule == "fixed":
            A_o = oracle.update_fixed(A64, G_o, cfg.alpha)
        else:
            A_o, S_o = oracle.update_adaptive(A64, np.zeros_like(A64), G_o, cfg.eta, b=bpar)
            assert rel_err(h.get_accum(n), S_o, np.linalg.norm(S_o)) <= 2 * TOL["f32"]
        A_g = Ad[n].cpu().numpy()
        assert rel_err(A_g, A_o, np.linalg.norm(A_o)) <= TOL["f32"]
        assert row_rel_err(A_g, A_o) <= 10 * TOL["f32"]
        for k in range(len(dims)):
            if k != n:
                assert np.array_equal(Ad[k].cpu().numpy(), A0[k])
        h.close()


@pytest.mark.parametrize("strategy", S)
@pytest.mark.parametrize("rule", ["adaptive", "fixed"])
def test_pw_trace_teacher_forced(strategy, rule):
    """four cyclic sweeps in ONE persistent launch: the traced batches, tables and updates of every
    iteration checked against the oracle from the traced state of that moment."""
    dims, R, B = (300, 130, 200), 50, 4096
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule=rule, row_sigma=1.0, noise=1e-2, seed=4, alpha=0.005,
                      eta=0.03)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, strategy, seed=11, fused=False, mode_major=True)
    assert h.path == "persistent"
    h.trace_start(12)
    h.sweep(4)
    recs = h.trace_read()
    assert len(recs) == 12 and [r["n"] for r in recs] == [0, 1, 2] * 4
    q0 = [h0[1] for h0 in oracle_tables(strategy, A0)]
    trace_check(X, dims, A0, recs, strategy, B, 11, rule, cfg, q0)
    for k in range(3):  # the final factors are the traced ones
        last = max(i for i, r in enumerate(recs) if r["n"] == k)
        assert np.array_equal(Ad[k].cpu().numpy(), recs[last]["A"])
    h.close()


def test_pw_rank_deficient_factor_tables():
    """Leverage tables of rank-deficient factors at R > 32 with I_n >= 2R (the tensor-core block inverse): a
    duplicated column makes a pivot fail the single-pivot rule inside an 8-pivot block, the kernel re-runs the
    pivot-by-pivot sweep from the Gram (reading R4(b): the pivot is skipped) and every rebuilt table equals the
    oracle's (QR with column pivoting, numerical rank R - 1).  alpha = 0: the factors stay rank-deficient."""
    dims, R, B = (152, 100, 90), 40, 512  # I_0 % 4 == 0: the persistent path gathers mode 0 in place
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule="fixed", row_sigma=1.0, noise=1e-2, seed=8, alpha=0.0)
    X, A0 = make_problem(cfg)
    for A in A0:
        A[:, 21] = A[:, 6]  # inside the block of pivots 16..23: the second of the pair fails
    Xd, Ad = to_dev(X, A0)
    for strategy in ("leverage", "block_leverage"):
        h = handle(cfg, Xd, Ad, strategy, seed=3, fused=False, mode_major=True)
        assert h.path == "persistent"
        h.trace_start(6)
        h.sweep(2)
        recs = h.trace_read()
        q0 = [t[1] for t in oracle_tables(strategy, A0)]
        trace_check(X, dims, A0, recs, strategy, B, 3, "fixed", cfg, q0)
        for k in range(3):
            assert np.array_equal(Ad[k].cpu().numpy(), A0[k])
        h.close()


def test_pw_random_order_and_schedule():
    """random mode order and a per-iteration fixed-step schedule in one launch."""
    dims, R, B = (200, 150, 100), 16, 1024
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule="fixed", row_sigma=1.0, noise=1e-2, seed=6)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "euclidean", seed=2, fused=False, mode_major=True)
    h.trace_start(9)
    h.sweep(3, order="random")
    recs = h.trace_read()
    modes = [oracle.random_mode(2, r, 3) for r in range(9)]
    assert [r["n"] for r in recs] == modes
    q0 = [t[1] for t in oracle_tables("euclidean", A0)]
    trace_check(X, dims, A0, recs, "euclidean", B, 2, "fixed", cfg, q0)
    al = 0.004 / (1.0 + np.arange(9)) ** 0.6
    h.trace_start(9)
    h.sweep(3, alphas=al)
    recs2 = h.trace_read()
    A1 = [a.copy() for a in A0]
    for r in recs:
        A1[r["n"]] = r["A"]
    q1 = list(q0)
    for r in recs:
        q1[r["n"]] = np.diff(np.concatenate([[0], r["cdf"]])).astype(np.uint64)
    trace_check(X, dims, A1, recs2, "euclidean", B, 2, "fixed", cfg, q1, alphas=al)
    h.close()


def test_pw_degenerate_table_stops():
    """a diverged step makes the next table non-finite: the launch stops and the status surfaces"""
    from paper_2103_04081_b200 import CPError

    cfg = synth.small((200, 100, 60), 8, dtype="f32", batch=512, rule="fixed", seed=1)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", fused=False, mode_major=True)
    assert h.path == "persistent"
    h.step(0, float("inf"))
    with pytest.raises(CPError, match="ENONFINITE|EDEGENERATE"):
        h.sync()
    h.close()


def test_pw_trace_two_units_per_cta():
    """a mode with more row units than CTAs (2600 rows = 163 units on 148 CTAs) over three traced sweeps: the
    second unit of a CTA re-reads its rows, the table prefix runs over several units per CTA"""
    dims, R, B = (2600, 40, 30), 16, 1024
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule="adaptive", row_sigma=1.0, noise=1e-2, seed=12, eta=0.03)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=13, fused=False, mode_major=True)
    assert h.path == "persistent"
    h.trace_start(9)
    h.sweep(3)
    recs = h.trace_read()
    assert [r["n"] for r in recs] == [0, 1, 2] * 3
    q0 = [t[1] for t in oracle_tables("leverage", A0)]
    trace_check(X, dims, A0, recs, "leverage", B, 13, "adaptive", cfg, q0)
    h.close()



def test_pw_falls_back_to_the_chain_when_not_coresident(monkeypatch):
    """a cooperative launch the device refuses (grid not co-resident, simulated by CPSGD_PW_FORCE_FALLBACK) runs the
    same steps on the kernel chain: same batches, results within the fp32 tolerance of the persistent run"""
    dims, R, B = (300, 130, 200), 20, 1024
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule="adaptive", row_sigma=1.0, noise=1e-2, seed=3, eta=0.03)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=5, fused=False, mode_major=True)
    assert h.path == "persistent"
    h.sweep(2)
    h.sync()
    ref = [a.cpu().numpy().astype(np.float64) for a in Ad]
    h.close()
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=5, fused=False, mode_major=True)
    monkeypatch.setenv("CPSGD_PW_FORCE_FALLBACK", "1")
    h.sweep(1)
    h.step(0)
    h.step(1)
    h.step(2)
    h.sync()
    monkeypatch.delenv("CPSGD_PW_FORCE_FALLBACK")
    assert h.path == "chain" and h.iter == 6
    for k in range(3):
        assert rel_err(Ad[k].cpu().numpy(), ref[k], np.linalg.norm(ref[k])) <= 1e-3
    h.close()


def test_pw_steps_host_optimistic_and_take_over():
    """cp_sgd_steps_host on the persistent path (whole cyclic sweeps): with host factors equal to the device copy the
    one launch runs the sweep (bitwise the device-path sweep of an identical handle); with changed host factors the
    launch does nothing (the flags say so), the changed factors are taken over with their tables rebuilt and the
    sweep runs -- the result equals a fresh handle started from those factors at the same iteration."""
    dims, R, B = (152, 100, 90), 40, 512
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule="fixed", row_sigma=1.0, noise=1e-2, seed=9, alpha=0.004)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=4, fused=False, mode_major=True)
    assert h.path == "persistent"
    host = [torch.from_numpy(a.copy()).pin_memory() for a in A0]
    h.steps_host(0, 3, host)
    _, Ar = to_dev(X, A0)
    ref = handle(cfg, Xd, Ar, "leverage", seed=4, fused=False, mode_major=True)
    ref.sweep(1)
    ref.sync()
    for k in range(3):
        assert np.array_equal(host[k].numpy(), Ar[k].cpu().numpy())
        assert np.array_equal(Ad[k].cpu().numpy(), Ar[k].cpu().numpy())
    ref.close()
    rng = np.random.default_rng(7)
    A1 = [host[k].numpy() * (1.0 + 0.05 * rng.standard_normal(A0[k].shape)).astype(np.float32) for k in range(3)]
    host = [torch.from_numpy(a.copy()).pin_memory() for a in A1]
    h.steps_host(0, 3, host)
    assert h.iter == 6
    _, Ar = to_dev(X, A1)
    ref = handle(cfg, Xd, Ar, "leverage", seed=4, fused=False, mode_major=True)
    ref.iter = 3
    ref.sweep(1)
    ref.sync()
    for k in range(3):
        a, b = host[k].numpy().astype(np.float64), Ar[k].cpu().numpy().astype(np.float64)
        assert np.linalg.norm(a - b) <= 1e-4 * np.linalg.norm(b)
    ref.close()
    h.close()


def test_pw_steps_host_refused_launch_takes_over(monkeypatch):
    """cp_sgd_steps_host's optimistic persistent launch refused (grid not co-resident, simulated): nothing runs in
    the optimistic call, the changed host factors are taken over and the sweep runs once on the kernel chain --
    equal to a fresh handle started from those factors at the same iteration."""
    dims, R, B = (152, 100, 90), 40, 512
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule="fixed", row_sigma=1.0, noise=1e-2, seed=9, alpha=0.004)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=4, fused=False, mode_major=True)
    assert h.path == "persistent"
    rng = np.random.default_rng(11)
    A1 = [(a * (1.0 + 0.05 * rng.standard_normal(a.shape))).astype(np.float32) for a in A0]
    host = [torch.from_numpy(a.copy()).pin_memory() for a in A1]
    monkeypatch.setenv("CPSGD_PW_FORCE_FALLBACK", "1")
    h.steps_host(0, 3, host)
    monkeypatch.delenv("CPSGD_PW_FORCE_FALLBACK")
    assert h.iter == 3 and h.path == "chain"
    _, Ar = to_dev(X, A1)
    ref = handle(cfg, Xd, Ar, "leverage", seed=4, fused=False, mode_major=True)
    ref.sweep(1)
    ref.sync()
    for k in range(3):
        a, b = host[k].numpy().astype(np.float64), Ar[k].cpu().numpy().astype(np.float64)
        assert np.linalg.norm(a - b) <= 1e-4 * np.linalg.norm(b)
    ref.close()
    h.close()


def test_pw_steps_host_packed_factors_one_transfer():
    """cp_sgd_steps_host with the factors back to back on both sides (views into one device block and one pinned host
    block): one transfer each way -- the same bits as the per-mode copies of separate buffers."""
    dims, R, B = (152, 100, 90), 40, 512
    cfg = synth.small(dims, R, dtype="f32", batch=B, rule="fixed", row_sigma=1.0, noise=1e-2, seed=9, alpha=0.004)
    X, A0 = make_problem(cfg)
    Xd = torch.from_numpy(X).to("cuda")
    flat = torch.empty(sum(a.size for a in A0), dtype=torch.float32, device="cuda")
    hflat = torch.empty(flat.numel(), dtype=torch.float32).pin_memory()
    Ad, host, o = [], [], 0
    for a in A0:
        Ad.append(flat[o:o + a.size].view(a.shape))
        host.append(hflat[o:o + a.size].view(a.shape))
        Ad[-1].copy_(torch.from_numpy(a))
        host[-1].copy_(torch.from_numpy(a))
        o += a.size
    h = handle(cfg, Xd, Ad, "leverage", seed=4, fused=False, mode_major=True)
    assert h.path == "persistent"
    h.steps_host(0, 3, host)
    h.steps_host(0, 3, host)
    _, As = to_dev(X, A0)
    ref = handle(cfg, Xd, As, "leverage", seed=4, fused=False, mode_major=True)
    hs = [torch.from_numpy(a.copy()).pin_memory() for a in A0]
    ref.steps_host(0, 3, hs)
    ref.steps_host(0, 3, hs)
    for k in range(3):
        assert np.array_equal(host[k].numpy(), hs[k].numpy())
    ref.close()
    h.close()
