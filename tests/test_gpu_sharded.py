"""Slab-sharded path on ONE GPU ("virtual shards"): P external-comm handles, each holding one
last-mode slab of X and its own factor replica; the test performs the exchanges (sum of the
partial-M buffers in rank order, copy of the owned rows) that NCCL performs on a real box.
Results must match the 1-GPU handle (and hence the oracle) -- same global batch every step."""
import numpy as np
import pytest

import synth
from gpu_helpers import handle, make_problem, rel_err, to_dev

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("strategy", ["leverage", "euclidean", "uniform", "block_leverage"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("mode_major", [True, False])
def test_virtual_shards_match_single_gpu(strategy, P, mode_major):
    from paper_2103_04081_b200 import CPSGD
    from paper_2103_04081_b200.parallel import slab_ranges

    dims = (20, 16, 12)
    cfg = synth.small(dims, 4, dtype="f64", batch=32, rule="fixed", seed=6, alpha=0.002, row_sigma=0.7)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h1 = handle(cfg, Xd, Ad, strategy, seed=5, fused=False, mode_major=mode_major)
    dev = torch.device("cuda:0")
    X3 = X.reshape(dims[::-1])  # C-order view of the first-index-fastest tensor: [i3][i2][i1]
    slabs = slab_ranges(dims[-1], P)
    hs, facs, keep = [], [], []
    for g, (lo, hi) in enumerate(slabs):
        Xg = torch.from_numpy(np.ascontiguousarray(X3[lo:hi]).ravel()).to(dev)
        Ag = [torch.from_numpy(a.copy()).to(dev) for a in A0]
        keep.append(Xg)
        facs.append(Ag)
        hs.append(CPSGD(Xg, dims, Ag, cfg.batch, sampler=strategy, rule="fixed", alpha=cfg.alpha, seed=5,
                        world_rank=g, world_size=P, slab=(lo, hi), external_comm=True, mode_major=mode_major,
                        fused=False))
    N = 3
    for it in range(3 * N):
        n = it % N
        h1.step(n, cfg.alpha)
        for h in hs:
            h.step_phase(n, 0, cfg.alpha)
        if n < N - 1:
            bufs = []
            for h in hs:
                b = torch.empty(h.exchange_count(n), dtype=torch.float64, device=dev)
                h.exchange_copy(n, b, False)
                bufs.append(b)
            torch.cuda.synchronize()
            tot = bufs[0].clone()
            for b in bufs[1:]:
                tot += b
            for h in hs:
                h.exchange_copy(n, tot, True)
        for h in hs:
            h.step_phase(n, 1, cfg.alpha)
        if n == N - 1:
            torch.cuda.synchronize()
            for g, (lo, hi) in enumerate(slabs):
                for gg in range(P):
                    if gg != g:
                        facs[gg][n][lo:hi].copy_(facs[g][n][lo:hi])
        for h in hs:
            h.step_phase(n, 2, cfg.alpha)
    torch.cuda.synchronize()
    import oracle

    fs, _, _ = oracle.run(X, A0, oracle.STRATEGIES[strategy], oracle.STEP_FIXED, cfg.batch, 3 * N, alpha=cfg.alpha,
                          seed=5)
    for g in range(P):
        for k in range(N):
            ref = Ad[k].cpu().numpy()
            assert rel_err(facs[g][k].cpu().numpy(), ref, np.linalg.norm(ref)) <= 1e-12
            # and the oracle's own run (not only the 1-GPU CUDA handle)
            assert rel_err(facs[g][k].cpu().numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-10
    # every replica drew the same batches: identical iteration counters
    assert all(h.iter == h1.iter == 3 * N for h in hs)
    for h in hs + [h1]:
        h.close()


# ------------------------------------------------------------------ stratified per-slab sampling (8(f).4)
def _oracle_stratified_run(X, dims, A0, strategy, B, seed, iters, alpha, lo):
    """Alg. 6 with the stratified sampler (reading R26): oracle.sample_stratified -> oracle.gradient ->
    oracle.update_fixed -> table rebuild of the updated mode (R9), cyclic modes"""
    import oracle

    st = oracle.STRATEGIES[strategy]
    A = [np.asarray(a, np.float64).copy() for a in A0]
    tabs = [oracle.build_table(st, a)[1:] for a in A]
    for r in range(iters):
        n = r % len(dims)
        idx, _, pj = oracle.sample_stratified(dims, n, st, B, tabs, seed, r, lo)
        G, _, _ = oracle.gradient(X, dims, A, n, st, B, idx, pj)
        A[n] = oracle.update_fixed(A[n], G, alpha)
        tabs[n] = oracle.build_table(st, A[n])[1:]
    return A


@pytest.mark.parametrize("strategy", ["leverage", "euclidean", "uniform"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("balanced", [False, True])
def test_virtual_shards_stratified_match_oracle(strategy, P, balanced):
    """P external-comm handles with CP_FLAG_STRATIFIED on one GPU: every rank's draws bit-exact with
    oracle.sample_stratified, each rank gathers exactly its stratum (B_g fibers, all in its slab), and three
    sweeps equal the oracle's stratified run; slabs equal or mass-balanced (cp_slice_sqnorms of the seeded
    tensor, checked against numpy, then parallel.balanced_slab_ranges)"""
    import oracle
    from paper_2103_04081_b200 import CPSGD
    from paper_2103_04081_b200.cpsgd import slice_sqnorms
    from paper_2103_04081_b200.parallel import balanced_slab_ranges, slab_bounds, slab_ranges

    dims = (20, 16, 12)
    cfg = synth.small(dims, 4, dtype="f64", batch=32, rule="fixed", seed=6, alpha=0.002, row_sigma=0.7)
    X, A0 = make_problem(cfg)
    dev = torch.device("cuda:0")
    X3 = X.reshape(dims[::-1])  # [i3][i2][i1]
    if balanced:
        e = slice_sqnorms(torch.from_numpy(X).to(dev), dims[-1]).cpu().numpy()
        np.testing.assert_allclose(e, (X3.reshape(dims[-1], -1) ** 2).sum(1), rtol=1e-12)
        slabs = balanced_slab_ranges(e, P)
    else:
        slabs = slab_ranges(dims[-1], P)
    lo = slab_bounds(slabs)
    hs, facs, keep = [], [], []
    for g, (a, b) in enumerate(slabs):
        Xg = torch.from_numpy(np.ascontiguousarray(X3[a:b]).ravel()).to(dev)
        Ag = [torch.from_numpy(x.copy()).to(dev) for x in A0]
        keep.append(Xg)
        facs.append(Ag)
        hs.append(CPSGD(Xg, dims, Ag, cfg.batch, sampler=strategy, rule="fixed", alpha=cfg.alpha, seed=5,
                        world_rank=g, world_size=P, slab=(a, b), external_comm=True, fused=False, stratified=True,
                        slab_bounds=lo))
    st = oracle.STRATEGIES[strategy]
    tabs = [oracle.build_table(st, np.asarray(x, np.float64))[1:] for x in A0]
    for n in range(2):  # the draws of modes n < N-1, every rank, bit-exact
        io, wo, _ = oracle.sample_stratified(dims, n, st, cfg.batch, tabs, 5, 0, lo)
        for h in hs:
            ig, wg = h.sample(n, 0)
            assert np.array_equal(ig.cpu().numpy(), io) and np.array_equal(wg.cpu().numpy(), wo)
        Bg = [cfg.batch // P + (1 if g < cfg.batch % P else 0) for g in range(P)]
        own = [int(((io[:, -1] >= a) & (io[:, -1] < b)).sum()) for a, b in slabs]
        assert own == Bg  # balanced owner-computes: rank g gathers exactly its stratum
    N = 3
    for it in range(3 * N):
        n = it % N
        for h in hs:
            h.step_phase(n, 0, cfg.alpha)
        if n < N - 1:
            bufs = []
            for h in hs:
                b = torch.empty(h.exchange_count(n), dtype=torch.float64, device=dev)
                h.exchange_copy(n, b, False)
                bufs.append(b)
            torch.cuda.synchronize()
            tot = bufs[0].clone()
            for b in bufs[1:]:
                tot += b
            for h in hs:
                h.exchange_copy(n, tot, True)
        for h in hs:
            h.step_phase(n, 1, cfg.alpha)
        if n == N - 1:
            torch.cuda.synchronize()
            for g, (a, b) in enumerate(slabs):
                for gg in range(P):
                    if gg != g:
                        facs[gg][n][a:b].copy_(facs[g][n][a:b])
        for h in hs:
            h.step_phase(n, 2, cfg.alpha)
    torch.cuda.synchronize()
    ref = _oracle_stratified_run(X, dims, A0, strategy, cfg.batch, 5, 3 * N, cfg.alpha, lo)
    for g in range(P):
        for k in range(N):
            assert rel_err(facs[g][k].cpu().numpy(), ref[k], np.linalg.norm(ref[k])) <= 1e-10
    for h in hs:
        h.close()


def test_stratified_refused_configs():
    from paper_2103_04081_b200 import CPSGD, CPError

    dims = (20, 16, 12)
    cfg = synth.small(dims, 4, dtype="f64", batch=32, rule="fixed", seed=6)
    X, A0 = make_problem(cfg)
    dev = torch.device("cuda:0")
    X3 = X.reshape(dims[::-1])
    Xg = torch.from_numpy(np.ascontiguousarray(X3[0:6]).ravel()).to(dev)
    Ag = [torch.from_numpy(x.copy()).to(dev) for x in A0]
    base = dict(rule="fixed", world_rank=0, world_size=2, slab=(0, 6), external_comm=True, fused=False,
                stratified=True)
    with pytest.raises(CPError, match="EINVAL"):  # external comm without the bounds
        CPSGD(Xg, dims, Ag, 32, sampler="leverage", **base)
    with pytest.raises(CPError, match="EINVAL"):  # block sampler
        CPSGD(Xg, dims, Ag, 32, sampler="block_leverage", slab_bounds=[0, 6, 12], **base)
    with pytest.raises(CPError, match="EINVAL"):  # bounds not matching this rank's slab
        CPSGD(Xg, dims, Ag, 32, sampler="leverage", slab_bounds=[0, 5, 12], **base)
    with pytest.raises(CPError, match="EINVAL"):  # batch < world
        CPSGD(Xg, dims, Ag, 1, sampler="leverage", slab_bounds=[0, 6, 12], **base)
