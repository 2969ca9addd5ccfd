"""Thin Python binding of libcpsgd.so (include/cpsgd.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels.  PyTorch supplies device
memory (the tensor X and the factors are borrowed torch CUDA tensors) and the stream.  There is
no CPU fallback: constructing a handle without the built library, or without a CUDA device,
raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcpsgd.so")

SAMPLERS = {"uniform": 0, "leverage": 1, "euclidean": 2, "block_leverage": 3, "block_euclidean": 4}
RULES = {"fixed": 0, "adaptive": 1, "als": 2}
ORDERS = {"cyclic": 0, "random": 1}
FLAG_MODE_MAJOR, FLAG_NO_GRAPH, FLAG_EXTERNAL_COMM, FLAG_NO_FUSED, FLAG_NO_WIDE, FLAG_NO_TC, FLAG_FUSED_CU8 = \
    0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40
FLAG_NO_PERSIST = 0x80
FLAG_STRATIFIED = 0x100
FLAG_REPLICA = 0x200
FLAG_FORCE_COMM = 0x400
FLAG_P2P = 0x800
KERNEL_NAMES = ["k_sample", "k_gather", "k_update_table", "k_table", "k_reduce_partials", "nccl", "k_fit",
                "k_sweep_fused", "k_gather_update", "k_zw_gamma", "k_gather_update_tc", "k_table_sample",
                "k_update_wide", "k_scores_wide", "k_sample_wide", "k_sweep_wide"]
STATUS = {0: "CP_OK", -1: "CP_EINVAL", -2: "CP_ERANGE", -3: "CP_EDEGENERATE", -4: "CP_ENOMEM", -5: "CP_ECUDA",
          -6: "CP_ENCCL", -7: "CP_ESTATE", -8: "CP_ENONFINITE"}

EXPORTS = ["cp_sgd_init", "cp_sgd_destroy", "cp_sgd_last_error", "cp_sgd_sample", "cp_sgd_step", "cp_sgd_sweep",
           "cp_fit", "cp_sgd_sync", "cp_sgd_steps_host", "cp_sgd_sweep_multi", "cp_sgd_step_phase", "cp_sgd_exchange_info",
           "cp_sgd_get_table", "cp_sgd_get_grad", "cp_sgd_get_accum", "cp_sgd_get_iter", "cp_sgd_set_iter",
           "cp_sgd_refresh_tables", "cp_sgd_get_launches", "cp_sgd_profile", "cp_sgd_profile_read",
           "cp_sgd_version", "cp_sgd_batch_max", "cp_sgd_debug_timers", "cp_sgd_exchange_copy", "cp_sgd_trace_layout",
           "cp_sgd_trace", "cp_sgd_trace_count", "cp_sgd_path", "cp_slice_sqnorms", "cp_nccl_unique_id", "cp_sgd_p2p_buffer",
           "cp_ipc_get_handle", "cp_sgd_p2p_open", "cp_sgd_p2p_peers"]


class CPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [
        ("order", C.c_int32), ("dims", C.POINTER(C.c_int64)), ("rank", C.c_int32), ("dtype", C.c_int32),
        ("X", C.c_void_p), ("factors", C.POINTER(C.c_void_p)), ("batch", C.c_int64),
        ("block_window", C.POINTER(C.c_int32)), ("sampler", C.c_int32), ("rule", C.c_int32),
        ("alpha", C.c_double), ("eta", C.c_double), ("b", C.c_double), ("eps", C.c_double),
        ("seed", C.c_uint64), ("stream", C.c_void_p), ("world_rank", C.c_int32), ("world_size", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("slab_begin", C.c_int64), ("slab_end", C.c_int64), ("flags", C.c_uint32),
        ("slab_bounds", C.POINTER(C.c_int64)),
    ]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libcpsgd.so (raises if it has not been built -- no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    P, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    L.cp_sgd_init.argtypes = [C.POINTER(Config), C.POINTER(C.c_void_p)]
    L.cp_sgd_destroy.argtypes = [P]
    L.cp_sgd_last_error.argtypes = [P]
    L.cp_sgd_last_error.restype = C.c_char_p
    L.cp_sgd_batch_max.argtypes = [P, i32, C.POINTER(C.c_int64)]
    L.cp_sgd_sample.argtypes = [P, i32, u64, P, P, C.POINTER(C.c_int64)]
    L.cp_sgd_step.argtypes = [P, i32, dbl]
    L.cp_sgd_sweep.argtypes = [P, i32, i32, P]
    L.cp_fit.argtypes = [P, C.POINTER(C.c_double)]
    L.cp_sgd_sync.argtypes = [P]
    L.cp_sgd_steps_host.argtypes = [P, i32, i32, dbl, P]
    L.cp_sgd_sweep_multi.argtypes = [P, i32, i32]
    L.cp_sgd_step_phase.argtypes = [P, i32, i32, dbl]
    L.cp_sgd_exchange_info.argtypes = [P, i32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64)]
    L.cp_sgd_get_table.argtypes = [P, i32, P, P, P]
    L.cp_sgd_get_grad.argtypes = [P, P, C.POINTER(C.c_int32), P]
    L.cp_sgd_get_accum.argtypes = [P, i32, P]
    L.cp_sgd_get_iter.argtypes = [P, C.POINTER(C.c_uint64)]
    L.cp_sgd_set_iter.argtypes = [P, u64]
    L.cp_sgd_refresh_tables.argtypes = [P]
    L.cp_sgd_get_launches.argtypes = [P, C.POINTER(C.c_uint64)]
    L.cp_sgd_profile.argtypes = [P, i32]
    L.cp_sgd_profile_read.argtypes = [P, i32, P, P, P, C.POINTER(C.c_int32)]
    L.cp_sgd_version.restype = C.c_char_p
    L.cp_sgd_debug_timers.argtypes = [P, P]
    L.cp_sgd_exchange_copy.argtypes = [P, i32, P, i32]
    L.cp_sgd_trace_layout.argtypes = [P, P]
    L.cp_sgd_trace.argtypes = [P, P, i64]
    L.cp_sgd_trace_count.argtypes = [P, C.POINTER(C.c_int64)]
    L.cp_sgd_path.argtypes = [P, C.POINTER(C.c_int32)]
    L.cp_slice_sqnorms.argtypes = [P, i32, i64, i64, P, P]
    L.cp_nccl_unique_id.argtypes = [P]
    L.cp_sgd_p2p_buffer.argtypes = [P, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
    L.cp_ipc_get_handle.argtypes = [P, P]
    L.cp_sgd_p2p_open.argtypes = [P, P]
    L.cp_sgd_p2p_peers.argtypes = [P, P]
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype if name in ("cp_sgd_last_error", "cp_sgd_version") else C.c_int
    _lib = L
    return L


def _dtype_code(t) -> int:
    import torch

    if t.dtype == torch.float32:
        return 0
    if t.dtype == torch.float64:
        return 1
    raise TypeError(f"unsupported dtype {t.dtype} (float32 / float64)")


class CPSGD:
    """Handle on one importance-sampled SGD chain (cp_sgd_t).

    X        : torch CUDA tensor holding the (local slab of the) dense tensor, first-index-fastest
               (a C-contiguous tensor of shape (I_N, ..., I_1) has exactly this layout)
    factors  : list of N torch CUDA tensors, I_n x R, contiguous, same dtype as X (updated in place)
    """

    def __init__(self, X, dims: Sequence[int], factors: List, batch: int, sampler: str = "leverage",
                 rule: str = "fixed", alpha: float = 0.01, eta: float = 0.05, b: float = 0.0, eps: float = 0.0,
                 seed: int = 0, stream=None, world_rank: int = 0, world_size: int = 1, nccl_id: bytes = None,
                 slab=None, mode_major: bool = True, block_window=None, graphs: bool = True,
                 external_comm: bool = False, fused: bool = True, wide: bool = True,
                 tc: bool = True, fused_cluster: int = 16, persist: bool = True, stratified: bool = False,
                 slab_bounds=None, replica: bool = False, force_comm: bool = False, p2p: bool = False):
        import torch

        L = load_library()
        if not X.is_cuda:
            raise ValueError("X must be a CUDA tensor (no CPU path exists)")
        self.N = len(dims)
        self.dims = [int(d) for d in dims]
        self.R = int(factors[0].shape[1])
        self.dtype = _dtype_code(X)
        for A, I in zip(factors, self.dims):
            if not (A.is_cuda and A.is_contiguous() and A.dtype == X.dtype and tuple(A.shape) == (I, self.R)):
                raise ValueError("factors must be contiguous CUDA tensors I_n x R of X's dtype")
        if not X.is_contiguous():
            raise ValueError("X must be contiguous")
        self._X, self._factors = X, list(factors)     # keep the borrowed buffers alive
        self._dims_arr = (C.c_int64 * self.N)(*self.dims)
        self._fac_arr = (C.c_void_p * self.N)(*[A.data_ptr() for A in factors])
        self._win_arr = None if block_window is None else (C.c_int32 * (self.N - 1))(*[int(w) for w in block_window])
        if stream is None:
            stream = torch.cuda.current_stream(X.device)
        self.stream = stream
        self._nccl_id = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
        flags = (FLAG_MODE_MAJOR if mode_major else 0) | (0 if graphs else FLAG_NO_GRAPH) | \
                (FLAG_EXTERNAL_COMM if external_comm else 0) | (0 if fused else FLAG_NO_FUSED) | \
                (0 if wide else FLAG_NO_WIDE) | (0 if tc else FLAG_NO_TC) | \
                (FLAG_FUSED_CU8 if fused_cluster == 8 else 0) | (0 if persist else FLAG_NO_PERSIST) | \
                (FLAG_STRATIFIED if stratified else 0) | (FLAG_REPLICA if replica else 0) | \
                (FLAG_FORCE_COMM if force_comm else 0) | (FLAG_P2P if p2p else 0)
        lo, hi = (0, self.dims[-1]) if slab is None else (int(slab[0]), int(slab[1]))
        cfg = Config(self.N, self._dims_arr, self.R, self.dtype, X.data_ptr(), self._fac_arr, int(batch),
                     self._win_arr, SAMPLERS[sampler], RULES[rule], float(alpha), float(eta), float(b), float(eps),
                     int(seed) & (2 ** 64 - 1), stream.cuda_stream, int(world_rank), int(world_size),
                     None if self._nccl_id is None else C.cast(self._nccl_id, C.c_void_p), lo, hi, flags,
                     None if slab_bounds is None else self._bounds_arr(slab_bounds))
        h = C.c_void_p()
        st = L.cp_sgd_init(C.byref(cfg), C.byref(h))
        if st != 0:
            raise CPError(st, L.cp_sgd_last_error(None).decode())
        self._h = h
        self._L = L
        self.batch = int(batch)
        self.sampler = sampler
        self.rule = rule
        self.slab = (lo, hi)
        self.world_size = world_size

    def _bounds_arr(self, bounds):
        self._bounds = (C.c_int64 * len(bounds))(*[int(b) for b in bounds])
        return C.cast(self._bounds, C.POINTER(C.c_int64))

    # -- plumbing -----------------------------------------------------------------------------
    def _chk(self, st):
        if st != 0:
            raise CPError(st, self._L.cp_sgd_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.cp_sgd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the hot path -----------------------------------------------------------------------------
    def sample(self, mode: int, it: int):
        """(idx int32 [B_eff, N-1], omega fp64 [B_eff]) on the device."""
        import torch

        bm = C.c_int64(0)
        self._chk(self._L.cp_sgd_batch_max(self._h, mode, C.byref(bm)))
        bmax = bm.value
        # the library writes on its own stream: allocate there (no fill kernel to race with), after
        # the caller's pending work
        self.stream.wait_stream(torch.cuda.current_stream(self._X.device))
        with torch.cuda.stream(self.stream):
            idx = torch.empty((bmax, self.N - 1), dtype=torch.int32, device=self._X.device)
            w = torch.empty(bmax, dtype=torch.float64, device=self._X.device)
        beff = C.c_int64(0)
        self._chk(self._L.cp_sgd_sample(self._h, mode, C.c_uint64(it), C.c_void_p(idx.data_ptr()),
                                        C.c_void_p(w.data_ptr()), C.byref(beff)))
        return idx[:beff.value], w[:beff.value]

    def batch_max(self, mode: int) -> int:
        bm = C.c_int64(0)
        self._chk(self._L.cp_sgd_batch_max(self._h, mode, C.byref(bm)))
        return bm.value

    def step(self, mode: int, alpha: float = -1.0):
        self._chk(self._L.cp_sgd_step(self._h, mode, float(alpha)))

    def step_phase(self, mode: int, phase: int, alpha: float = -1.0):
        self._chk(self._L.cp_sgd_step_phase(self._h, mode, phase, float(alpha)))

    def exchange_info(self, mode: int):
        buf, cnt, rb, re = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64()
        self._chk(self._L.cp_sgd_exchange_info(self._h, mode, C.byref(buf), C.byref(cnt), C.byref(rb), C.byref(re)))
        return buf.value, cnt.value, rb.value, re.value

    def p2p_buffer(self):
        """(device pointer, bytes) of this replica's symmetric exchange buffer (CP_FLAG_P2P)"""
        buf, nb = C.c_void_p(), C.c_int64()
        self._chk(self._L.cp_sgd_p2p_buffer(self._h, C.byref(buf), C.byref(nb)))
        return buf.value, nb.value

    def p2p_ipc_handle(self) -> bytes:
        """64-byte cudaIpcMemHandle of the exchange buffer, to send to the other ranks"""
        out = C.create_string_buffer(64)
        buf, _ = self.p2p_buffer()
        st = self._L.cp_ipc_get_handle(C.c_void_p(buf), out)
        if st != 0:
            raise CPError(st, "cp_ipc_get_handle")
        return bytes(out.raw)

    def p2p_open(self, handles):
        """map every rank's exchange buffer from its IPC handle (rank order, 64 bytes each)"""
        blob = b"".join(bytes(hd) for hd in handles)
        self._chk(self._L.cp_sgd_p2p_open(self._h, C.create_string_buffer(blob, len(blob))))

    def p2p_peers(self, ptrs):
        """register device pointers of every rank's exchange buffer (rank order) addressable here"""
        arr = (C.c_void_p * len(ptrs))(*[int(x) for x in ptrs])
        self._chk(self._L.cp_sgd_p2p_peers(self._h, arr))

    def exchange_count(self, mode: int) -> int:
        """elements of the phase-0 exchange buffer of `mode` (slabs: partial M, R x I_n; replicas: the rank's
        chunk sum of M, ceil(I_n/128) x R x 128)"""
        return int(self.exchange_info(mode)[1])

    def exchange_copy(self, mode: int, buf, to_lib: bool):
        """copy the phase-0 exchange buffer (exchange_count(mode) elements) to / from a torch CUDA tensor"""
        self._chk(self._L.cp_sgd_exchange_copy(self._h, mode, C.c_void_p(buf.data_ptr()), 1 if to_lib else 0))

    @staticmethod
    def sweep_multi(handles, nsweeps: int = 1):
        """nsweeps cyclic sweeps of every handle in ONE launch, one cluster per chain;
        the handles must share the fused geometry (dtype, dims, R)."""
        hs = list(handles)
        arr = (C.c_void_p * len(hs))(*[h._h for h in hs])
        hs[0]._chk(hs[0]._L.cp_sgd_sweep_multi(arr, len(hs), int(nsweeps)))

    def sweep(self, nsweeps: int = 1, order: str = "cyclic", alphas=None):
        arr = None
        if alphas is not None:
            a = np.ascontiguousarray(alphas, dtype=np.float64)
            assert a.size == nsweeps * self.N
            arr = a.ctypes.data_as(C.c_void_p)
        self._chk(self._L.cp_sgd_sweep(self._h, int(nsweeps), ORDERS[order], arr))

    def steps_host(self, first_mode: int, nsteps: int, factors_host: list, alpha: float = -1.0):
        """factors_host: list of N host tensors/arrays (pinned torch tensors recommended), updated in place."""
        ptrs = []
        for A in factors_host:
            ptrs.append(A.data_ptr() if hasattr(A, "data_ptr") else A.ctypes.data)
        arr = (C.c_void_p * self.N)(*ptrs)
        self._chk(self._L.cp_sgd_steps_host(self._h, int(first_mode), int(nsteps), float(alpha), arr))

    def fit(self) -> float:
        out = C.c_double(0.0)
        self._chk(self._L.cp_fit(self._h, C.byref(out)))
        return out.value

    def sync(self):
        self._chk(self._L.cp_sgd_sync(self._h))

    # -- parity / debug hooks -----------------------------------------------------------------------
    def get_table(self, mode: int):
        I = self.dims[mode]
        q = np.zeros(I, dtype=np.uint64)
        p = np.zeros(I, dtype=np.float64)
        T = C.c_uint64(0)
        self._chk(self._L.cp_sgd_get_table(self._h, mode, q.ctypes.data_as(C.c_void_p), C.byref(T),
                                           p.ctypes.data_as(C.c_void_p)))
        return q, int(T.value), p

    def get_grad(self):
        dt = np.float64 if self.dtype == 1 else np.float32
        m = C.c_int32(-1)
        self._chk(self._L.cp_sgd_get_grad(self._h, None, C.byref(m), None))
        G = np.zeros((self.dims[m.value], self.R), dtype=dt)
        Gam = np.zeros((self.R, self.R), dtype=dt)
        self._chk(self._L.cp_sgd_get_grad(self._h, G.ctypes.data_as(C.c_void_p), C.byref(m),
                                          Gam.ctypes.data_as(C.c_void_p)))
        return G, m.value, Gam

    def get_accum(self, mode: int):
        dt = np.float64 if self.dtype == 1 else np.float32
        S = np.zeros((self.dims[mode], self.R), dtype=dt)
        self._chk(self._L.cp_sgd_get_accum(self._h, mode, S.ctypes.data_as(C.c_void_p)))
        return S

    @property
    def iter(self) -> int:
        r = C.c_uint64(0)
        self._chk(self._L.cp_sgd_get_iter(self._h, C.byref(r)))
        return int(r.value)

    @iter.setter
    def iter(self, r: int):
        self._chk(self._L.cp_sgd_set_iter(self._h, C.c_uint64(r)))

    def refresh_tables(self):
        self._chk(self._L.cp_sgd_refresh_tables(self._h))

    @property
    def launches(self) -> int:
        n = C.c_uint64(0)
        self._chk(self._L.cp_sgd_get_launches(self._h, C.byref(n)))
        return int(n.value)

    @property
    def path(self) -> str:
        """'fused' (k_sweep_fused), 'persistent' (k_sweep_wide) or 'chain' (kernel chain / graph)"""
        v = C.c_int32(0)
        self._chk(self._L.cp_sgd_path(self._h, C.byref(v)))
        return {1: "fused", 2: "persistent"}.get(v.value, "chain")

    def trace_start(self, cap: int):
        """record the batches (and resulting factor / accumulator / table of the updated mode) of the
        next `cap` SGD iterations run by a persistent kernel; read them with trace_read()"""
        import torch

        lay = (C.c_int64 * 7)()
        self._chk(self._L.cp_sgd_trace_layout(self._h, lay))
        self._trace_layout = list(lay)
        self._trace_buf = torch.zeros(int(cap) * lay[0], dtype=torch.uint8, device=self._X.device)
        torch.cuda.synchronize(self._X.device)
        self._chk(self._L.cp_sgd_trace(self._h, C.c_void_p(self._trace_buf.data_ptr()), int(cap)))

    def trace_read(self):
        """list of per-iteration dicts {n, r, beff, idx, w, A, S, cdf} (numpy, host)"""
        self.sync()
        cnt = C.c_int64(0)
        self._chk(self._L.cp_sgd_trace_count(self._h, C.byref(cnt)))
        stride, o_idx, o_w, o_A, o_S, o_cdf, o_meta = self._trace_layout
        raw = self._trace_buf.cpu().numpy()
        dt = np.float64 if self.dtype == 1 else np.float32
        bm = max(self.batch_max(k) for k in range(self.N))
        out = []
        for s in range(cnt.value):
            rec = raw[s * stride:(s + 1) * stride]
            meta = rec[o_meta:o_meta + 32].view(np.int64)
            n, r, beff = int(meta[0]), int(meta[1]), int(meta[2])
            I = self.dims[n]
            out.append(dict(n=n, r=r, beff=beff,
                            idx=rec[o_idx:o_idx + 4 * bm * (self.N - 1)].view(np.int32).reshape(bm, self.N - 1)[:beff].copy(),
                            w=rec[o_w:o_w + 8 * bm].view(np.float64)[:beff].copy(),
                            A=rec[o_A:o_A + I * self.R * np.dtype(dt).itemsize].view(dt).reshape(I, self.R).copy(),
                            S=rec[o_S:o_S + I * self.R * np.dtype(dt).itemsize].view(dt).reshape(I, self.R).copy(),
                            cdf=rec[o_cdf:o_cdf + 8 * I].view(np.uint64).copy()))
        return out

    def trace_stop(self):
        self._chk(self._L.cp_sgd_trace(self._h, None, 0))

    def debug_timers(self):
        out = (C.c_longlong * (4096 + 8 * 160 * 32))()
        self._chk(self._L.cp_sgd_debug_timers(self._h, out))
        return list(out)

    def profile(self, on: bool):
        self._chk(self._L.cp_sgd_profile(self._h, 1 if on else 0))

    def profile_read(self):
        cap = 16
        ids = (C.c_int32 * cap)()
        tot = (C.c_double * cap)()
        cnt = (C.c_int64 * cap)()
        n = C.c_int32(0)
        self._chk(self._L.cp_sgd_profile_read(self._h, cap, ids, tot, cnt, C.byref(n)))
        return {KERNEL_NAMES[ids[i]]: (tot[i], int(cnt[i])) for i in range(n.value)}


def slice_sqnorms(X, nslices: int, stream=None):
    """cp_slice_sqnorms: fp64 squared norms of the nslices last-mode slices of the CUDA tensor X (a
    torch tensor; marshalling only -- the sums run in the library's kernels)."""
    import torch

    L = load_library()
    if not X.is_cuda or not X.is_contiguous():
        raise ValueError("X must be a contiguous CUDA tensor")
    out = torch.empty(int(nslices), dtype=torch.float64, device=X.device)
    s = torch.cuda.current_stream(X.device) if stream is None else stream
    st = L.cp_slice_sqnorms(X.data_ptr(), _dtype_code(X), int(nslices), X.numel() // int(nslices), out.data_ptr(),
                            s.cuda_stream)
    if st != 0:
        raise CPError(st, "cp_slice_sqnorms")
    return out


def nccl_unique_id() -> bytes:
    """cp_nccl_unique_id: a fresh 128-byte ncclUniqueId from the library's own NCCL"""
    L = load_library()
    buf = C.create_string_buffer(128)
    st = L.cp_nccl_unique_id(buf)
    if st != 0:
        raise CPError(st, "cp_nccl_unique_id")
    return bytes(buf.raw)

