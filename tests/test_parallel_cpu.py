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
