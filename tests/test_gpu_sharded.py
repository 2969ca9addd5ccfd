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
                b = torch.empty(cfg.rank * dims[n], dtype=torch.float64, device=dev)
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
