"""paper_2501_15126_b200 -- thin Python binding of libperm (include/perm.h).

B200-native sparse permanent (Elbek & Kaya, arXiv 2501.15126): every step of
the hot path runs in libperm (C++ planner + NVRTC-generated sm_100a kernels +
fixed sm_100a reduction kernels).  This module only marshals arguments; it
never computes a permanent itself and has no CPU fallback.

Functions mirror the C ABI names (perm_plan, perm_compute, perm_free, ...);
`Plan` is a small owning wrapper.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._abi import MODE, ORDER, PERM_CCS, PERM_CRS, STATUS, perm_opts, perm_plan_info, perm_result

__all__ = ["PermError", "Plan", "Comm", "perm_plan", "perm_compute", "perm_compute_ex", "perm_compute_shard",
           "perm_compute_async", "perm_compute_partial", "perm_plan_export", "perm_plan_import",
           "perm_probe_fp64_peak",
           "perm_fold", "perm_free", "perm_structural_rank", "perm_order", "perm_partition",
           "perm_alg2_launch_parameters", "dense_to_ccs", "dense_to_crs", "perm_version"]


class PermError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _abi.lib().perm_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st: int, where: str):
    if st != 0:
        raise PermError(st, where)


def _i32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _f64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def dense_to_ccs(A):
    """Dense -> (cptrs, rids, cvals) (Sec. II); complex dense -> complex cvals."""
    A = np.asarray(A)
    cpx = np.iscomplexobj(A)
    A = A.astype(np.complex128 if cpx else np.float64)
    n = A.shape[0]
    ptr, idx, val = [0], [], []
    for j in range(n):
        rows = np.nonzero(A[:, j])[0]
        idx.extend(rows.tolist())
        val.extend(A[rows, j].tolist())
        ptr.append(len(idx))
    return np.array(ptr, np.int32), np.array(idx, np.int32), np.array(val, np.complex128 if cpx else np.float64)


def dense_to_crs(A):
    return dense_to_ccs(np.asarray(A).T)


def make_opts(mode="auto", device=0, stream=None, chunk_log2=0, block_log2=0, task_chunks=0,
              gr_ratio=0.0, hybrid_c=0, threads_per_block=0, no_device=False, factor_cols=0,
              min_blocks=0, zero_skip=0, autotune=0, rank=0, world=0, reseed_log2=0, nccl_comm=None,
              cache_dir=None) -> perm_opts:
    o = perm_opts()
    o.rank = rank
    o.world = world
    o.reseed_log2 = reseed_log2
    o.nccl_comm = nccl_comm.handle if isinstance(nccl_comm, Comm) else nccl_comm
    o.cache_dir = cache_dir.encode() if isinstance(cache_dir, str) else cache_dir
    o.autotune = autotune
    o.factor_cols = factor_cols
    o.min_blocks = min_blocks
    o.zero_skip = zero_skip
    o.mode = MODE[mode] if isinstance(mode, str) else int(mode)
    o.device = int(device)
    o.cuda_stream = stream
    o.chunk_log2 = chunk_log2
    o.block_log2 = block_log2
    o.task_chunks = task_chunks
    o.gr_ratio = gr_ratio
    o.hybrid_c = hybrid_c
    o.threads_per_block = threads_per_block
    o.no_device = 1 if no_device else 0
    return o


def perm_plan(n, fmt, ptr, idx, val, ordering="auto", opts: perm_opts | None = None) -> int:
    L = _abi.lib()
    ptr_a, p_ptr = _i32(ptr)
    idx_a, p_idx = _i32(idx)
    h = ctypes.c_void_p()
    o = ORDER[ordering] if isinstance(ordering, str) else int(ordering)
    if np.iscomplexobj(val):   # complex permanent: interleaved (re, im)
        val_a, p_val = _f64(np.ascontiguousarray(np.asarray(val, np.complex128)).view(np.float64))
        st = L.perm_plan_complex(n, fmt, p_ptr, p_idx, p_val, o, ctypes.byref(opts or make_opts()),
                                 ctypes.byref(h))
        _check(st, "perm_plan_complex")
        return h.value
    val_a, p_val = _f64(val)
    if opts is None:
        st = L.perm_plan(n, fmt, p_ptr, p_idx, p_val, o, ctypes.byref(h))
    else:
        st = L.perm_plan_ex(n, fmt, p_ptr, p_idx, p_val, o, ctypes.byref(opts), ctypes.byref(h))
    _check(st, "perm_plan")
    return h.value


def perm_compute(h) -> float:
    return _abi.lib().perm_compute(h)


def perm_compute_ex(h) -> perm_result:
    r = perm_result()
    _check(_abi.lib().perm_compute_ex(h, ctypes.byref(r)), "perm_compute_ex")
    return r


def perm_compute_shard(h, rank: int, world: int) -> perm_result:
    r = perm_result()
    _check(_abi.lib().perm_compute_shard(h, rank, world, ctypes.byref(r)), "perm_compute_shard")
    return r


def perm_compute_shard_async(h, rank: int, world: int, d_partial: int):
    _check(_abi.lib().perm_compute_shard_async(h, rank, world, ctypes.c_void_p(d_partial)),
           "perm_compute_shard_async")


def perm_fold(h, shards) -> perm_result:
    arr = (perm_result * len(shards))(*shards)
    out = perm_result()
    _check(_abi.lib().perm_fold(h, arr, len(shards), ctypes.byref(out)), "perm_fold")
    return out


def perm_fold_async(h, d_partials: int, world: int, d_out: int):
    _check(_abi.lib().perm_fold_async(h, ctypes.c_void_p(d_partials), world, ctypes.c_void_p(d_out)),
           "perm_fold_async")


def perm_compute_async(h, d_out: int):
    _check(_abi.lib().perm_compute_async(h, ctypes.c_void_p(d_out)), "perm_compute_async")


def perm_compute_partial(h, rank: int, world: int):
    buf = (ctypes.c_double * 2)()
    _check(_abi.lib().perm_compute_partial(h, rank, world, buf), "perm_compute_partial")
    return buf[0], buf[1]


def perm_plan_export(h) -> bytes:
    L = _abi.lib()
    sz = ctypes.c_size_t(0)
    _check(L.perm_plan_export(h, None, ctypes.byref(sz)), "perm_plan_export")
    buf = ctypes.create_string_buffer(sz.value)
    _check(L.perm_plan_export(h, buf, ctypes.byref(sz)), "perm_plan_export")
    return buf.raw[: sz.value]


def perm_plan_import(blob: bytes, opts: perm_opts | None = None) -> int:
    h = ctypes.c_void_p()
    _check(_abi.lib().perm_plan_import(blob, len(blob), ctypes.byref(opts or make_opts()), ctypes.byref(h)),
           "perm_plan_import")
    return h.value


def perm_probe_fp64_peak(device: int = 0):
    """Measured FP64 lane-ops/s of `device` and the best kernel ms (perm.h)."""
    v, ms = ctypes.c_double(), ctypes.c_double()
    _check(_abi.lib().perm_probe_fp64_peak(device, ctypes.byref(v), ctypes.byref(ms)), "perm_probe_fp64_peak")
    return v.value, ms.value


class Comm:
    """NCCL communicator owned by libperm (perm_comm_init); rank 0's 128-byte
    unique id must reach every rank first (comm_unique_id + any transport)."""

    def __init__(self, world: int, rank: int, uid: bytes, device: int = 0):
        h = ctypes.c_void_p()
        _check(_abi.lib().perm_comm_init(world, rank, uid, device, ctypes.byref(h)), "perm_comm_init")
        self.handle, self.world, self.rank = h.value, world, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(_abi.lib().perm_comm_unique_id(buf), "perm_comm_unique_id")
        return buf.raw

    def close(self):
        if getattr(self, "handle", None):
            _check(_abi.lib().perm_comm_destroy(self.handle), "perm_comm_destroy")
            self.handle = None


def perm_free(h):
    if h:
        _abi.lib().perm_free(h)


def perm_version() -> str:
    return _abi.lib().perm_version().decode()


def perm_structural_rank(n, fmt, ptr, idx, val) -> int:
    ptr_a, p_ptr = _i32(ptr)
    idx_a, p_idx = _i32(idx)
    val_a, p_val = _f64(val)
    r = _abi.lib().perm_structural_rank(n, fmt, p_ptr, p_idx, p_val)
    if r < 0:
        raise PermError(1, "perm_structural_rank")
    return r


def perm_order(n, fmt, ptr, idx, val, ordering="permanent"):
    ptr_a, p_ptr = _i32(ptr)
    idx_a, p_idx = _i32(idx)
    val_a, p_val = _f64(val)
    rp = np.zeros(n, np.int32)
    cp = np.zeros(n, np.int32)
    st = _abi.lib().perm_order(n, fmt, p_ptr, p_idx, p_val, ORDER[ordering],
                               rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                               cp.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    _check(st, "perm_order")
    return rp.tolist(), cp.tolist()


def perm_partition(n, cptrs, rids, gr_ratio=16.0, sms=148):
    cp_a, p_cp = _i32(cptrs)
    ri_a, p_ri = _i32(rids)
    k, c = ctypes.c_int(), ctypes.c_int()
    _check(_abi.lib().perm_partition(n, p_cp, p_ri, gr_ratio, sms, ctypes.byref(k), ctypes.byref(c)),
           "perm_partition")
    return k.value, c.value


def perm_alg2_launch_parameters(tau: int, n: int, cap: int = 4096):
    buf = (ctypes.c_uint64 * (3 * cap))()
    cnt = _abi.lib().perm_alg2_launch_parameters(tau, n, buf, cap)
    if cnt < 0:
        raise PermError(1, "perm_alg2_launch_parameters")
    return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(min(cnt, cap))]


class Plan:
    """Owning wrapper of a perm_plan_t."""

    def __init__(self, n, fmt, ptr, idx, val, ordering="auto", **opts):
        self.n = int(n)
        self.is_complex = bool(np.iscomplexobj(val))
        self._opts = make_opts(**opts)   # kept alive: cache_dir / comm pointers
        self.handle = perm_plan(self.n, fmt, ptr, idx, val, ordering, self._opts)

    @classmethod
    def from_blob(cls, blob: bytes, **opts):
        """Plan from a perm_plan_export blob (no search, no NVRTC)."""
        self = cls.__new__(cls)
        self._opts = make_opts(**opts)
        self.handle = perm_plan_import(blob, self._opts)
        self.n = self.info["n"]
        self.is_complex = self.info["mode"] == 4
        return self

    def export(self) -> bytes:
        return perm_plan_export(self.handle)

    def compute_async(self, d_out: int):
        perm_compute_async(self.handle, d_out)

    def compute_partial(self, rank: int, world: int):
        re, im = perm_compute_partial(self.handle, rank, world)
        return complex(re, im) if self.is_complex else re

    @classmethod
    def from_dense(cls, A, ordering="auto", fmt=PERM_CCS, **opts):
        A = np.asarray(A)
        A = A.astype(np.complex128 if np.iscomplexobj(A) else np.float64)
        ptr, idx, val = dense_to_ccs(A) if fmt == PERM_CCS else dense_to_crs(A)
        return cls(A.shape[0], fmt, ptr, idx, val, ordering, **opts)

    def compute(self):
        r = self.compute_ex()
        return r.complex_value() if self.is_complex else r.value

    def compute_ex(self) -> perm_result:
        return perm_compute_ex(self.handle)

    def exact(self) -> int | None:
        return self.compute_ex().exact()

    def shard(self, rank: int, world: int) -> perm_result:
        return perm_compute_shard(self.handle, rank, world)

    def fold(self, shards) -> perm_result:
        return perm_fold(self.handle, shards)

    def shard_async(self, rank: int, world: int, d_partial: int):
        perm_compute_shard_async(self.handle, rank, world, d_partial)

    def fold_async(self, d_partials: int, world: int, d_out: int):
        perm_fold_async(self.handle, d_partials, world, d_out)

    def shard_range(self, rank: int, world: int):
        """(first_task, ntasks, g_begin, g_end) of shard `rank` of `world`."""
        v = [ctypes.c_uint64() for _ in range(4)]
        _check(_abi.lib().perm_shard_range(self.handle, rank, world, *[ctypes.byref(x) for x in v]),
               "perm_shard_range")
        return tuple(x.value for x in v)

    def fold_host(self, partials) -> float:
        arr = np.ascontiguousarray(np.asarray(partials, dtype=np.float64))
        return _abi.lib().perm_fold_host(self.handle, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                         len(arr))

    def last_timing(self):
        """(sweep_ms, reduce_ms) of the last launch, from the plan's CUDA events."""
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(_abi.lib().perm_last_timing(self.handle, ctypes.byref(a), ctypes.byref(b)), "perm_last_timing")
        return a.value, b.value

    @property
    def partial_bytes(self) -> int:
        return _abi.lib().perm_partial_bytes(self.handle)

    @property
    def info(self) -> dict:
        i = perm_plan_info()
        _check(_abi.lib().perm_plan_get_info(self.handle, ctypes.byref(i)), "perm_plan_get_info")
        return i.as_dict()

    @property
    def source(self) -> str:
        return _abi.lib().perm_plan_source(self.handle).decode()

    def cubin(self) -> bytes:
        L = _abi.lib()
        sz = ctypes.c_size_t(0)
        _check(L.perm_plan_cubin(self.handle, None, ctypes.byref(sz)), "perm_plan_cubin")
        buf = ctypes.create_string_buffer(sz.value)
        _check(L.perm_plan_cubin(self.handle, buf, ctypes.byref(sz)), "perm_plan_cubin")
        return buf.raw[: sz.value]

    def task_partials(self, cap: int = 1 << 24):
        """Per-warp-task partial sums of the last compute/shard call."""
        L = _abi.lib()
        pb = self.partial_bytes
        cnt = ctypes.c_uint64()
        first = ctypes.c_uint64()
        _check(L.perm_debug_task_partials(self.handle, None, 0, ctypes.byref(cnt), ctypes.byref(first)),
               "perm_debug_task_partials")
        # query count with cap 0 returns 0; ask again with the real cap
        buf = np.zeros(cap * (pb // 8), np.uint64 if (pb == 16 and not self.is_complex) else np.float64)
        _check(L.perm_debug_task_partials(self.handle, buf.ctypes.data, cap, ctypes.byref(cnt),
                                          ctypes.byref(first)), "perm_debug_task_partials")
        c = cnt.value
        if self.is_complex:
            return first.value, buf[:2 * c].view(np.complex128).copy()
        if pb == 16:
            lo = buf[0:2 * c:2].astype(object)
            hi = buf[1:2 * c:2].astype(object)
            vals = [(int(h) << 64) | int(l) for l, h in zip(lo, hi)]
            return first.value, [v - (1 << 128) if v >> 127 else v for v in vals]
        return first.value, buf[:c].copy()

    def close(self):
        if getattr(self, "handle", None):
            perm_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
