"""Host-side plumbing of the slab-sharded path.

The tensor is split along its LAST mode into contiguous slabs, one per rank.  Every rank holds
replicated factors and tables and draws the same global batch (same Philox counters).  One SGD
iteration of mode n is three library phases (cp_sgd_step_phase) with one exchange:
  n <  N-1 : phase 0 (local fibers -> partial M) ; all-reduce(M) ; phase 1 (update) ; phase 2
  n == N-1 : phase 0 (local rows of every fiber) ; phase 1 (update of the owned rows) ;
             broadcast every rank's owned rows ; phase 2 (table refresh)
With an internal NCCL communicator the library performs these exchanges itself (cp_sgd_step);
`ShardedRunner` performs them through a `torch.distributed` process group instead (external-comm
handles), which is also how the host logic is tested on CPU with the gloo backend.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def slab_ranges(I_last: int, world: int) -> List[Tuple[int, int]]:
    """contiguous, near-equal slabs [lo, hi) of the last mode's index range, rank order."""
    if world < 1 or I_last < world:
        raise ValueError("need 1 <= world <= I_last")
    base, extra = divmod(I_last, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def balanced_slab_ranges(weights, world: int, max_len: int = None) -> List[Tuple[int, int]]:
    """Mass-balanced contiguous slabs (SURVEY 8(e) mitigation 2): rank-order ranges [lo, hi) of the last mode
    whose total `weights` (e.g. the slice energies ||X(:, ..., :, i)||^2 from cp_slice_sqnorms, the proxy of
    the sampling mass the last factor converges to) are as equal as the contiguity allows.  Boundary g is
    the index whose cumulative weight is closest to g/world of the total, kept inside the feasible range
    (every slab non-empty and at most max_len long, so each rank's slab fits its memory).  With stratified
    sampling (CP_FLAG_STRATIFIED) equal-mass slabs make the equal per-rank strata close to proportional
    allocation, which never has a larger variance than unstratified sampling."""
    w = [float(x) for x in weights]
    n = len(w)
    if world < 1 or n < world:
        raise ValueError("need 1 <= world <= number of slices")
    if any(x < 0 or x != x for x in w):
        raise ValueError("weights must be finite and >= 0")
    cap = n if max_len is None else int(max_len)
    if cap * world < n:
        raise ValueError("max_len too small: the slabs cannot cover every slice")
    cum = [0.0]
    for x in w:
        cum.append(cum[-1] + x)
    tot = cum[-1]
    bounds = [0]
    for g in range(1, world):
        lo_ok = max(bounds[-1] + 1, n - (world - g) * cap)  # later slabs must still fit
        hi_ok = min(bounds[-1] + cap, n - (world - g))      # later slabs non-empty
        if tot > 0:
            target = tot * g / world
            b = min(max(lo_ok, 1), hi_ok)
            best, bd = b, abs(cum[b] - target)
            for c in range(lo_ok, hi_ok + 1):  # plain scan: the closest feasible cumulative weight
                d = abs(cum[c] - target)
                if d < bd:
                    best, bd = c, d
            b = best
        else:
            b = min(max(lo_ok, (n * g) // world), hi_ok)
        bounds.append(b)
    bounds.append(n)
    return [(bounds[g], bounds[g + 1]) for g in range(world)]


def slab_bounds(ranges) -> List[int]:
    """[lo_0, lo_1, ..., lo_{P-1}, hi_{P-1}]: the cp_sgd_config.slab_bounds array of contiguous ranges"""
    out = [int(ranges[0][0])]
    for (lo, hi), nxt in zip(ranges, list(ranges[1:]) + [None]):
        if nxt is not None and int(nxt[0]) != int(hi):
            raise ValueError("slab ranges are not contiguous")
        out.append(int(hi))
    return out


def owned_fibers(idx_last, lo: int, hi: int):
    """mask of sampled fibers whose last-mode index falls in this rank's slab (owner computes)."""
    return (idx_last >= lo) & (idx_last < hi)


class ShardedRunner:
    """Drives one external-comm handle per rank.  `handle` needs step_phase(mode, phase, alpha),
    exchange_copy(mode, buf, to_lib) and factor tensors; `group` is a torch.distributed group."""

    def __init__(self, handle, factors: Sequence, dims: Sequence[int], rank: int, world: int, group=None,
                 device=None):
        import torch

        self.h = handle
        self.factors = list(factors)
        self.dims = [int(d) for d in dims]
        self.N = len(self.dims)
        self.R = int(self.factors[0].shape[1])
        self.rank, self.world, self.group = rank, world, group
        self.slabs = slab_ranges(self.dims[-1], world)
        self.device = device if device is not None else self.factors[0].device
        self.dtype = self.factors[0].dtype
        self._buf = {}
        self.torch = torch

    def _exchange_sum(self, n: int):
        import torch.distributed as dist

        # the library's exchange-buffer size (the wide path: the rank's chunk sum, ceil(I_n/128) x R x 128)
        count = self.h.exchange_count(n) if hasattr(self.h, "exchange_count") else self.R * self.dims[n]
        key = (n, count)
        if key not in self._buf:
            self._buf[key] = self.torch.empty(count, dtype=self.dtype, device=self.device)
        buf = self._buf[key]
        self.h.exchange_copy(n, buf, False)
        self.sync()
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
        self._order_after_collective()
        self.h.exchange_copy(n, buf, True)

    def _exchange_rows(self, n: int):
        import torch.distributed as dist

        self.sync()
        A = self.factors[n]
        for r, (lo, hi) in enumerate(self.slabs):
            rows = A[lo:hi].contiguous()
            dist.broadcast(rows, src=r, group=self.group)
            if r != self.rank:
                A[lo:hi].copy_(rows)
        self._order_after_collective()

    def _order_after_collective(self):
        """the collectives and copies above ran on torch's current stream; the library's next phase
        runs on the handle's stream: make that stream wait for them (no-op on CPU / gloo)"""
        hs = getattr(self.h, "stream", None)
        if hs is not None and self.torch.cuda.is_available() and hasattr(hs, "wait_stream"):
            hs.wait_stream(self.torch.cuda.current_stream(hs.device))

    def sync(self):
        if hasattr(self.h, "sync"):
            self.h.sync()

    def step(self, n: int, alpha: float = -1.0):
        self.h.step_phase(n, 0, alpha)
        if n < self.N - 1:
            self._exchange_sum(n)
        self.h.step_phase(n, 1, alpha)
        if n == self.N - 1:
            self._exchange_rows(n)
        self.h.step_phase(n, 2, alpha)

    def sweep(self, nsweeps: int, alpha: float = -1.0):
        for _ in range(nsweeps):
            for n in range(self.N):
                self.step(n, alpha)


def p2p_connect(handle, group=None):
    """Map every rank's CP_FLAG_P2P exchange buffer into this process (one call per rank, collective over
    `group`): the 64-byte IPC handles are all-gathered through torch.distributed (rank order) and opened by
    the library (cp_sgd_p2p_open).  `handle` needs p2p_ipc_handle() and p2p_open(list)."""
    import torch.distributed as dist

    mine = handle.p2p_ipc_handle()
    world = dist.get_world_size(group)
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    handle.p2p_open(allh)
    return allh

