"""Multi-rank host logic of the slab-sharded path on CPU: world_size 2 over the gloo backend.

`ShardedRunner` (product host plumbing) drives, on each rank, a stand-in handle whose three
phases are computed by the oracle on that rank's slab -- partial M over the fibers the rank owns,
the update of the owned rows -- and performs the exchanges (all-reduce of M, broadcast of owned
rows) through torch.distributed.  The result must equal the single-process oracle run.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2103_04081_b200.parallel import ShardedRunner, owned_fibers, slab_ranges


def test_slab_ranges():
    assert slab_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert slab_ranges(4000, 8)[-1] == (3500, 4000)
    with pytest.raises(ValueError):
        slab_ranges(3, 4)


def test_owned_fibers_partition():
    idx = np.array([0, 3, 4, 9, 7])
    masks = [owned_fibers(idx, lo, hi) for lo, hi in slab_ranges(10, 3)]
    assert (sum(m.astype(int) for m in masks) == 1).all()


class OracleShardHandle:
    """stand-in for an external-comm library handle: phases computed by the oracle on this
    rank's view; the exchange buffer layout is the library's [R][I_local]."""

    def __init__(self, X, dims, factors, strategy, B, seed, rank, world, alpha):
        self.X, self.dims, self.N = X, list(dims), len(dims)
        self.f = factors                        # torch CPU tensors (shared with the runner)
        self.st = oracle.STRATEGIES[strategy]
        self.B, self.seed, self.alpha = B, seed, alpha
        self.lo, self.hi = slab_ranges(dims[-1], world)[rank]
        self.r = 0
        self.tables = [oracle.build_table(self.st, A.numpy()) for A in self.f]

    def step_phase(self, n, phase, alpha=-1.0):
        A = [a.numpy() for a in self.f]
        if phase == 0:
            tq = [(t[1], t[2]) for t in self.tables]
            idx, w, pj = oracle.sample(self.dims, n, self.st, self.B, tq, self.seed, self.r)
            _, self.Gam, Mfull = oracle.gradient(self.X, self.dims, A, n, self.st, self.B, idx, pj)
            if n < self.N - 1:
                own = owned_fibers(idx[:, -1], self.lo, self.hi)
                _, _, Mown = oracle.gradient(self.X, self.dims, A, n, self.st, self.B, idx[own], pj[own]) \
                    if own.any() else (None, None, np.zeros_like(Mfull))
                self.M = Mown
            else:
                self.M = Mfull[self.lo:self.hi]      # this rank's rows only
        elif phase == 1:
            rows = slice(0, self.dims[n]) if n < self.N - 1 else slice(self.lo, self.hi)
            G = A[n][rows] @ self.Gam - self.M
            self.f[n][rows] = torch.from_numpy(oracle.update_fixed(A[n][rows], G, self.alpha))
        else:
            self.tables[n] = oracle.build_table(self.st, self.f[n].numpy())
            self.r += 1

    def exchange_copy(self, n, buf, to_lib):
        if to_lib:
            self.M = buf.numpy().reshape(self.M.shape[1], self.M.shape[0]).T.copy()
        else:
            buf.copy_(torch.from_numpy(np.ascontiguousarray(self.M.T).ravel()))


def _worker(rank, world, port, strategy, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.small((7, 6, 8), 3, dtype="f64", batch=12, rule="fixed", seed=4, alpha=0.002)
    X = synth.tensor(cfg)
    A0 = synth.init_factors(cfg, X)
    facs = [torch.from_numpy(a.copy()) for a in A0]
    h = OracleShardHandle(X, cfg.dims, facs, strategy, cfg.batch, 11, rank, world, cfg.alpha)
    runner = ShardedRunner(h, facs, cfg.dims, rank, world)
    runner.sweep(4)
    out[rank] = [f.numpy().copy() for f in facs]
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("strategy", ["leverage", "euclidean", "uniform"])
def test_sharded_runner_gloo_matches_single_process(strategy):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), strategy, out), nprocs=world, join=True)
    cfg = synth.small((7, 6, 8), 3, dtype="f64", batch=12, rule="fixed", seed=4, alpha=0.002)
    X = synth.tensor(cfg)
    A0 = synth.init_factors(cfg, X)
    ref, _, _ = oracle.run(X, A0, oracle.STRATEGIES[strategy], oracle.STEP_FIXED, cfg.batch, 12, alpha=cfg.alpha,
                           seed=11)
    for r in range(world):
        for k in range(3):
            np.testing.assert_allclose(out[r][k], ref[k], rtol=1e-11, atol=1e-13)


def test_balanced_slab_ranges_properties():
    """contiguous rank-order cover, non-empty slabs, max_len respected, every interior boundary's cumulative
    weight within one slice weight of its target g/P of the total, and on lognormal slice weights (the
    survey's heavy-tailed rows) a smaller max/mean slab mass than equal-length slabs"""
    from paper_2103_04081_b200.parallel import balanced_slab_ranges, slab_bounds

    rng = np.random.default_rng(3)
    for P in (2, 4, 8):
        w = np.exp(rng.standard_normal(400) * 1.5)
        r = balanced_slab_ranges(w, P)
        b = slab_bounds(r)
        assert b[0] == 0 and b[-1] == 400 and all(hi > lo for lo, hi in r)
        cum = np.concatenate([[0.0], np.cumsum(w)])
        for g in range(1, P):
            assert abs(cum[b[g]] - cum[-1] * g / P) <= w.max()
        mass = np.array([w[lo:hi].sum() for lo, hi in r])
        eq = np.array([w[lo:hi].sum() for lo, hi in slab_ranges(400, P)])
        assert mass.max() / mass.mean() <= eq.max() / eq.mean()
        rc = balanced_slab_ranges(w, P, max_len=400 // P + 5)
        assert all(hi - lo <= 400 // P + 5 for lo, hi in rc) and slab_bounds(rc)[-1] == 400
    with pytest.raises(ValueError):
        balanced_slab_ranges(np.ones(10), 3, max_len=3)
    assert balanced_slab_ranges(np.zeros(10), 3) == [(0, 3), (3, 6), (6, 10)]


class OracleStratifiedShardHandle(OracleShardHandle):
    """the stand-in handle with stratified draws (oracle.sample_stratified, reading R26): rank g's own
    fibers are exactly its stratum"""

    def __init__(self, *a, bounds=None, **kw):
        super().__init__(*a, **kw)
        self.bounds = bounds

    def step_phase(self, n, phase, alpha=-1.0):
        if phase != 0:
            return super().step_phase(n, phase, alpha)
        A = [a.numpy() for a in self.f]
        tq = [(t[1], t[2]) for t in self.tables]
        idx, w, pj = oracle.sample_stratified(self.dims, n, self.st, self.B, tq, self.seed, self.r, self.bounds)
        _, self.Gam, Mfull = oracle.gradient(self.X, self.dims, A, n, self.st, self.B, idx, pj)
        if n < self.N - 1:
            own = owned_fibers(idx[:, -1], self.lo, self.hi)
            _, _, self.M = oracle.gradient(self.X, self.dims, A, n, self.st, self.B, idx[own], pj[own])
        else:
            self.M = Mfull[self.lo:self.hi]


def _worker_strat(rank, world, port, out):
    from paper_2103_04081_b200.parallel import slab_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.small((7, 6, 8), 3, dtype="f64", batch=12, rule="fixed", seed=4, alpha=0.002)
    X = synth.tensor(cfg)
    A0 = synth.init_factors(cfg, X)
    facs = [torch.from_numpy(a.copy()) for a in A0]
    h = OracleStratifiedShardHandle(X, cfg.dims, facs, "leverage", cfg.batch, 11, rank, world, cfg.alpha,
                                    bounds=slab_bounds(slab_ranges(8, world)))
    runner = ShardedRunner(h, facs, cfg.dims, rank, world)
    runner.sweep(4)
    out[rank] = [f.numpy().copy() for f in facs]
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_runner_gloo_stratified():
    """world 2 over gloo with stratified draws: both replicas equal a single-process stratified run"""
    from paper_2103_04081_b200.parallel import slab_bounds

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_strat, args=(world, _free_port(), out), nprocs=world, join=True)
    cfg = synth.small((7, 6, 8), 3, dtype="f64", batch=12, rule="fixed", seed=4, alpha=0.002)
    X = synth.tensor(cfg)
    A = [np.asarray(a, np.float64).copy() for a in synth.init_factors(cfg, X)]
    st = oracle.LEVERAGE
    lo = slab_bounds(slab_ranges(8, world))
    tabs = [oracle.build_table(st, a)[1:] for a in A]
    for r in range(12):
        n = r % 3
        idx, _, pj = oracle.sample_stratified(cfg.dims, n, st, cfg.batch, tabs, 11, r, lo)
        G, _, _ = oracle.gradient(X, cfg.dims, A, n, st, cfg.batch, idx, pj)
        A[n] = oracle.update_fixed(A[n], G, cfg.alpha)
        tabs[n] = oracle.build_table(st, A[n])[1:]
    for r in range(world):
        for k in range(3):
            np.testing.assert_allclose(out[r][k], A[k], rtol=1e-11, atol=1e-13)


class _StubP2P:
    def __init__(self, rank):
        self.rank = rank
        self.opened = None

    def p2p_ipc_handle(self):
        return bytes([self.rank + 1]) * 64

    def p2p_open(self, handles):
        self.opened = list(handles)


def _worker_p2p(rank, world, port, out):
    from paper_2103_04081_b200.parallel import p2p_connect

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = _StubP2P(rank)
    p2p_connect(h)
    out[rank] = h.opened
    dist.barrier()
    dist.destroy_process_group()


def test_p2p_connect_gathers_handles_in_rank_order():
    """host logic of the peer-memory exchange setup (CP_FLAG_P2P): every rank opens every rank's 64-byte IPC
    handle, in rank order (world 3 over gloo)"""
    world = 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_p2p, args=(world, _free_port(), out), nprocs=world, join=True)
    want = [bytes([g + 1]) * 64 for g in range(world)]
    for r in range(world):
        assert out[r] == want
