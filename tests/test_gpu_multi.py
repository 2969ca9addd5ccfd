"""Multi-rank code paths of the library on ONE GPU (VERDICT r01 "multi-GPU readiness").

* The library's own NCCL calls: a world_size == 1 handle forced onto the multi-rank path
  (CP_FLAG_FORCE_COMM) with a 1-rank communicator from cp_nccl_unique_id -- slab sharding
  (ncclAllReduce of M for modes n < N-1, ncclBroadcast of the owned rows of A^(N-1), ncclAllReduce of the
  fit partials) and whole-tensor replicas (CP_FLAG_REPLICA: ncclAllReduce of the chunk sums), run by
  cp_sgd_step / cp_sgd_sweep (direct and graph-captured) against the oracle's Alg. 6/7 run.
* Replicas with a batch split (BASELINE C4 at 2-8 GPUs): P external-comm replica handles on one GPU,
  rank g gathering the wide path's chunks g, g + P, ...; the test sums the ranks' chunk sums (what
  ncclAllReduce does) -- every rank's factors equal the single-GPU handle's and the oracle's.
No two handles ever wait on one another inside a kernel: each phase runs to completion on its own.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import TOL, handle, make_problem, oracle_step, rel_err, row_rel_err, to_dev

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()


@pytest.mark.parametrize("strategy", ["leverage", "euclidean", "uniform"])
@pytest.mark.parametrize("graphs", [False, True])
def test_force_comm_sharded_runs_nccl(strategy, graphs):
    from paper_2103_04081_b200.cpsgd import nccl_unique_id

    cfg = synth.CONFIGS["C1"]
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, strategy, seed=3, fused=False, force_comm=True, nccl_id=nccl_unique_id(),
               graphs=graphs)
    assert h.path == "chain"
    h.sweep(2)
    for n in range(3):
        h.step(n, cfg.alpha)
    h.sync()
    fs, _, _ = oracle.run(X, A0, oracle.STRATEGIES[strategy], oracle.STEP_FIXED, cfg.batch, 9, alpha=cfg.alpha, seed=3)
    for k in range(3):
        assert rel_err(Ad[k].cpu().numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-10
    assert abs(h.fit() - oracle.fit(X, fs)) <= 1e-10  # the fit partials went through ncclAllReduce
    h.close()


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_force_comm_replica_runs_nccl(dt):
    from paper_2103_04081_b200.cpsgd import nccl_unique_id

    if dt == "f64":
        cfg = synth.small((40, 30, 24), 6, dtype="f64", batch=96, rule="adaptive", eta=0.05, seed=2)
    else:
        cfg = synth.small((300, 130, 200), 20, dtype="f32", batch=1024, rule="adaptive", eta=0.03, seed=2)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    h = handle(cfg, Xd, Ad, "leverage", seed=4, fused=False, replica=True, force_comm=True, nccl_id=nccl_unique_id())
    assert h.path == "chain"
    if dt == "f64":
        h.sweep(3)
        h.sync()
        fs, _, _ = oracle.run(X, A0, oracle.LEVERAGE, oracle.STEP_ADAPTIVE, cfg.batch, 9, eta=cfg.eta, seed=4)
        for k in range(3):
            assert rel_err(Ad[k].cpu().numpy(), fs[k], np.linalg.norm(fs[k])) <= 1e-10
    else:  # fp32: one step per mode from the seeded state against the oracle's step
        h.close()
        for n in range(3):
            Xd, Ad = to_dev(X, A0)
            h = handle(cfg, Xd, Ad, "leverage", seed=4, fused=False, replica=True, force_comm=True,
                       nccl_id=nccl_unique_id())
            h.iter = 7 + n
            _, _, G_o, Gam_o, M_o, _ = oracle_step(X, cfg.dims, A0, n, "leverage", cfg.batch, 4, 7 + n)
            h.step(n)
            G_g, _, _ = h.get_grad()
            A64 = np.asarray(A0[n], np.float64)
            assert rel_err(G_g, G_o, np.linalg.norm(A64 @ Gam_o) + np.linalg.norm(M_o)) <= TOL["f32"]
            h.close()
        return
    h.close()


def _replica_run(cfg, X, A0, strategy, P, seed, iters, rule_kw):
    """P external-comm replica handles on one GPU; returns every rank's factors after `iters` cyclic steps"""
    from paper_2103_04081_b200 import CPSGD

    dev = torch.device("cuda:0")
    Xd = torch.from_numpy(X).to(dev)
    hs, facs = [], []
    for g in range(P):
        Ag = [torch.from_numpy(np.ascontiguousarray(a).copy()).to(dev) for a in A0]
        facs.append(Ag)
        hs.append(CPSGD(Xd, cfg.dims, Ag, cfg.batch, sampler=strategy, seed=seed, world_rank=g, world_size=P,
                        external_comm=True, replica=True, fused=False, **rule_kw))
    N = len(cfg.dims)
    for it in range(iters):
        n = it % N
        for h in hs:
            h.step_phase(n, 0)
        bufs = []
        for h in hs:
            b = torch.empty(h.exchange_count(n), dtype=Xd.dtype, device=dev)
            h.exchange_copy(n, b, False)
            bufs.append(b)
        torch.cuda.synchronize()
        tot = bufs[0].clone()
        for b in bufs[1:]:
            tot += b  # rank order (the allreduce's job)
        for h in hs:
            h.exchange_copy(n, tot, True)
        for h in hs:
            h.step_phase(n, 1)
        for h in hs:
            h.step_phase(n, 2)
    torch.cuda.synchronize()
    out = [[a.cpu().numpy() for a in Ag] for Ag in facs]
    for h in hs:
        h.close()
    return out


@pytest.mark.parametrize("strategy", ["leverage", "euclidean", "block_leverage", "uniform"])
@pytest.mark.parametrize("P", [2, 3])
def test_virtual_replicas_batch_split_match_single_gpu_and_oracle(strategy, P):
    cfg = synth.small((40, 30, 24), 6, dtype="f64", batch=96, rule="fixed", alpha=0.002, seed=5)
    X, A0 = make_problem(cfg)
    outs = _replica_run(cfg, X, A0, strategy, P, 6, 9, dict(rule="fixed", alpha=cfg.alpha))
    Xd, Ad = to_dev(X, A0)
    h1 = handle(cfg, Xd, Ad, strategy, seed=6, fused=False, persist=False)
    h1.sweep(3)
    h1.sync()
    fs, _, _ = oracle.run(X, A0, oracle.STRATEGIES[strategy], oracle.STEP_FIXED, cfg.batch, 9, alpha=cfg.alpha, seed=6)
    for g in range(P):
        for k in range(3):
            assert np.array_equal(outs[g][k], outs[0][k])  # the replicas stay bitwise identical
            ref = Ad[k].cpu().numpy()
            assert rel_err(outs[g][k], ref, np.linalg.norm(ref)) <= 1e-12   # = 1 GPU up to the sum order of M
            assert rel_err(outs[g][k], fs[k], np.linalg.norm(fs[k])) <= 1e-10  # = the oracle
    h1.close()


def test_virtual_replicas_f32_tcgen05_one_step():
    """fp32 replicas on the tcgen05 wide path (C4 shape in miniature, ragged tiles): one step per mode from
    the seeded state equals the oracle's step within the fp32 tolerance, on every rank"""
    cfg = synth.small((300, 130, 200), 20, dtype="f32", batch=1024, rule="adaptive", eta=0.03, seed=8)
    X, A0 = make_problem(cfg)
    for n in range(3):
        from paper_2103_04081_b200 import CPSGD

        P = 2
        dev = torch.device("cuda:0")
        Xd = torch.from_numpy(X).to(dev)
        hs, facs = [], []
        for g in range(P):
            Ag = [torch.from_numpy(a.copy()).to(dev) for a in A0]
            facs.append(Ag)
            h = CPSGD(Xd, cfg.dims, Ag, cfg.batch, sampler="leverage", rule="adaptive", eta=cfg.eta, seed=9,
                      world_rank=g, world_size=P, external_comm=True, replica=True, fused=False)
            h.iter = 3 + n
            hs.append(h)
        for h in hs:
            h.step_phase(n, 0)
        bufs = []
        for h in hs:
            b = torch.empty(h.exchange_count(n), dtype=torch.float32, device=dev)
            h.exchange_copy(n, b, False)
            bufs.append(b)
        torch.cuda.synchronize()
        tot = bufs[0] + bufs[1]
        for h in hs:
            h.exchange_copy(n, tot, True)
            h.step_phase(n, 1)
            h.step_phase(n, 2)
        torch.cuda.synchronize()
        _, _, G_o, Gam_o, M_o, _ = oracle_step(X, cfg.dims, A0, n, "leverage", cfg.batch, 9, 3 + n)
        A64 = np.asarray(A0[n], np.float64)
        A_o, _ = oracle.update_adaptive(A64, np.zeros_like(A64), G_o, cfg.eta)
        scale = np.linalg.norm(A64 @ Gam_o) + np.linalg.norm(M_o)
        band = np.abs(G_o) <= 10 * TOL["f32"] * scale / np.sqrt(G_o.size)  # b = 0: eta sign(G) (gpu_helpers)
        for g in range(P):
            A_g = facs[g][n].cpu().numpy().astype(np.float64)
            assert np.linalg.norm(np.where(band, 0.0, A_g - A_o)) <= TOL["f32"] * np.linalg.norm(A_o)
            assert row_rel_err(np.where(band, A_o, A_g), A_o) <= 10 * TOL["f32"]
            assert np.array_equal(facs[g][n].cpu().numpy(), facs[0][n].cpu().numpy())
        for h in hs:
            h.close()


def test_replica_refused_configs():
    from paper_2103_04081_b200 import CPError

    cfg = synth.small((40, 30, 24), 6, dtype="f64", batch=96, rule="fixed", seed=5)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    base = dict(world_rank=0, world_size=2, external_comm=True, replica=True, fused=False)
    with pytest.raises(CPError, match="EINVAL"):
        handle(cfg, Xd, Ad, "leverage", wide=False, **base)
    with pytest.raises(CPError, match="EINVAL"):
        handle(cfg, Xd, Ad, "leverage", stratified=True, slab_bounds=[0, 12, 24], **base)
    with pytest.raises(CPError, match="EINVAL"):  # fp32 tcgen05 chunks of 32 fibers: B = 32 is one chunk < P
        cfg32 = synth.small((40, 30, 24), 6, dtype="f32", batch=32, rule="fixed", seed=5)
        X32, A32 = make_problem(cfg32)
        Xd32, Ad32 = to_dev(X32, A32)
        handle(cfg32, Xd32, Ad32, "leverage", **base)


# ------------------------------------------------------------- replicas over peer memory (CP_FLAG_P2P)
def _p2p_run(cfg, X, A0, strategy, P, seed, iters, rule_kw):
    """P replica handles exchanging M through each other's symmetric buffers (addressable directly: one
    process, one GPU), all on ONE stream so every rank's phase 0 (publish) completes before any rank's
    phase 1 (peer reads) starts -- no kernel ever waits on another running kernel"""
    from paper_2103_04081_b200 import CPSGD

    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    Xd = torch.from_numpy(X).to(dev)
    hs, facs = [], []
    for g in range(P):
        Ag = [torch.from_numpy(np.ascontiguousarray(a).copy()).to(dev) for a in A0]
        facs.append(Ag)
        hs.append(CPSGD(Xd, cfg.dims, Ag, cfg.batch, sampler=strategy, seed=seed, world_rank=g, world_size=P,
                        replica=True, p2p=True, fused=False, stream=stream, **rule_kw))
    bufs = [h.p2p_buffer()[0] for h in hs]
    for h in hs:
        h.p2p_peers(bufs)
    N = len(cfg.dims)
    for it in range(iters):
        n = it % N
        for ph in range(3):
            for h in hs:
                h.step_phase(n, ph)
    torch.cuda.synchronize()
    out = [[a.cpu().numpy() for a in Ag] for Ag in facs]
    for h in hs:
        h.close()
    return out


@pytest.mark.parametrize("strategy", ["leverage", "euclidean", "uniform"])
@pytest.mark.parametrize("P", [2, 3])
def test_p2p_replicas_match_single_gpu_and_oracle(strategy, P):
    cfg = synth.small((40, 30, 24), 6, dtype="f64", batch=96, rule="fixed", alpha=0.002, seed=5)
    X, A0 = make_problem(cfg)
    outs = _p2p_run(cfg, X, A0, strategy, P, 6, 12, dict(rule="fixed", alpha=cfg.alpha))  # > 2 epochs per parity
    Xd, Ad = to_dev(X, A0)
    h1 = handle(cfg, Xd, Ad, strategy, seed=6, fused=False, persist=False)
    h1.sweep(4)
    h1.sync()
    fs, _, _ = oracle.run(X, A0, oracle.STRATEGIES[strategy], oracle.STEP_FIXED, cfg.batch, 12, alpha=cfg.alpha,
                          seed=6)
    for g in range(P):
        for k in range(3):
            assert np.array_equal(outs[g][k], outs[0][k])  # the same bytes on every rank (rank-order sum)
            ref = Ad[k].cpu().numpy()
            assert rel_err(outs[g][k], ref, np.linalg.norm(ref)) <= 1e-12
            assert rel_err(outs[g][k], fs[k], np.linalg.norm(fs[k])) <= 1e-10
    h1.close()


def test_p2p_replicas_f32_adaptive_trajectory_equals_nccl_style_sum():
    """fp32 tcgen05 replicas: the peer-memory exchange gives the same factors as the caller-summed
    (external-comm) exchange -- both sum the ranks' chunk sums in rank order"""
    cfg = synth.small((300, 130, 200), 20, dtype="f32", batch=1024, rule="adaptive", eta=0.03, seed=8)
    X, A0 = make_problem(cfg)
    a = _p2p_run(cfg, X, A0, "leverage", 2, 9, 6, dict(rule="adaptive", eta=cfg.eta))
    b = _replica_run(cfg, X, A0, "leverage", 2, 9, 6, dict(rule="adaptive", eta=cfg.eta))
    for g in range(2):
        for k in range(3):
            assert np.array_equal(a[g][k], b[g][k])


def test_p2p_api_errors_and_ipc_handle():
    from paper_2103_04081_b200 import CPError

    cfg = synth.small((40, 30, 24), 6, dtype="f64", batch=96, rule="fixed", seed=5)
    X, A0 = make_problem(cfg)
    Xd, Ad = to_dev(X, A0)
    with pytest.raises(CPError, match="EINVAL"):  # P2P without replicas
        handle(cfg, Xd, Ad, "leverage", world_rank=0, world_size=2, external_comm=True, p2p=True, fused=False)
    h = handle(cfg, Xd, Ad, "leverage", world_rank=0, world_size=2, replica=True, p2p=True, fused=False)
    with pytest.raises(CPError, match="ESTATE"):  # peers not registered yet
        h.step_phase(0, 0)
    buf, nbytes = h.p2p_buffer()
    assert buf and nbytes > 4096
    assert len(h.p2p_ipc_handle()) == 64
    with pytest.raises(CPError, match="EINVAL"):  # entry world_rank must be the handle's own buffer
        h.p2p_peers([buf + 4096, buf])
    h.close()
    h2 = handle(cfg, Xd, Ad, "leverage", fused=False)
    with pytest.raises(CPError, match="ESTATE"):
        h2.p2p_buffer()
    h2.close()
