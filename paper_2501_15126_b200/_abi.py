"""ctypes mirror of include/perm.h (argument marshalling only).

Loads the in-tree libperm.so; raises ImportError loudly if it is missing --
there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libperm.so")

PERM_CCS, PERM_CRS = 0, 1
ORDER = {"none": 0, "degree": 1, "permanent": 2, "auto": 3}
MODE = {"auto": 0, "reg": 1, "hybrid": 2, "int01": 3}
STATUS = {0: "PERM_OK", 1: "PERM_EINVAL", 2: "PERM_ERANGE", 3: "PERM_ENOMEM", 4: "PERM_ECUDA",
          5: "PERM_ENVRTC", 6: "PERM_ENCCL", 7: "PERM_ESPILL"}


class perm_opts(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("device", ctypes.c_int), ("cuda_stream", ctypes.c_void_p),
                ("chunk_log2", ctypes.c_int), ("block_log2", ctypes.c_int), ("task_chunks", ctypes.c_int),
                ("gr_ratio", ctypes.c_double), ("hybrid_c", ctypes.c_int),
                ("threads_per_block", ctypes.c_int), ("no_device", ctypes.c_int),
                ("factor_cols", ctypes.c_int), ("min_blocks", ctypes.c_int), ("zero_skip", ctypes.c_int),
                ("autotune", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int),
                ("reseed_log2", ctypes.c_int), ("reserved0", ctypes.c_int), ("nccl_comm", ctypes.c_void_p),
                ("cache_dir", ctypes.c_char_p)]


class perm_result(ctypes.Structure):
    _fields_ = [("value", ctypes.c_double), ("exact_lo", ctypes.c_uint64), ("exact_hi", ctypes.c_uint64),
                ("exact_valid", ctypes.c_int), ("world", ctypes.c_int), ("rank", ctypes.c_int),
                ("products", ctypes.c_uint64), ("sweep_ms", ctypes.c_double), ("reduce_ms", ctypes.c_double),
                ("value_im", ctypes.c_double), ("steps", ctypes.c_uint64), ("seconds", ctypes.c_double),
                ("w_plan", ctypes.c_double), ("k", ctypes.c_int), ("c", ctypes.c_int), ("b", ctypes.c_int),
                ("mode", ctypes.c_int), ("K", ctypes.c_int), ("reserved_r", ctypes.c_int)]

    def complex_value(self) -> complex:
        return complex(self.value, self.value_im)

    def exact(self):
        if not self.exact_valid:
            return None
        v = (self.exact_hi << 64) | self.exact_lo
        return v - (1 << 128) if v >> 127 else v


class perm_plan_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("nnz", ctypes.c_int), ("mode", ctypes.c_int), ("ordering", ctypes.c_int),
                ("singular", ctypes.c_int), ("struct_rank", ctypes.c_int), ("k", ctypes.c_int),
                ("c", ctypes.c_int), ("B", ctypes.c_int), ("U", ctypes.c_int), ("M", ctypes.c_int),
                ("K", ctypes.c_int), ("swept_order", ctypes.c_int), ("tasks", ctypes.c_uint64), ("reg_rows", ctypes.c_int), ("tier_rows", ctypes.c_int),
                ("seed_rows", ctypes.c_int), ("levels", ctypes.c_int), ("w_plan", ctypes.c_double),
                ("w_alg1", ctypes.c_double), ("block", ctypes.c_int), ("grid", ctypes.c_int),
                ("blocks_per_sm", ctypes.c_int), ("sms", ctypes.c_int), ("regs_per_thread", ctypes.c_int),
                ("local_bytes", ctypes.c_int), ("smem_bytes", ctypes.c_int), ("plan_ms", ctypes.c_double),
                ("codegen_ms", ctypes.c_double), ("nvrtc_ms", ctypes.c_double), ("cubin_cached", ctypes.c_int), ("plan_cached", ctypes.c_int),
                ("row_perm", ctypes.c_int * 64), ("col_perm", ctypes.c_int * 64),
                ("autotune_ms", ctypes.c_double), ("nvrtc_cpu_ms", ctypes.c_double), ("disk_cached", ctypes.c_int),
                ("candidates_compiled", ctypes.c_int)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            if name in ("row_perm", "col_perm"):
                v = list(v)[: self.n]
            d[name] = v
        return d


EXPORTS = ["perm_plan", "perm_plan_ex", "perm_compute", "perm_compute_ex", "perm_compute_shard",
           "perm_compute_shard_async", "perm_fold", "perm_fold_async", "perm_partial_bytes",
           "perm_debug_task_partials", "perm_last_timing", "perm_plan_get_info", "perm_plan_source", "perm_plan_cubin",
           "perm_free", "perm_last_error", "perm_version", "perm_structural_rank", "perm_order",
           "perm_partition", "perm_alg2_launch_parameters", "perm_shard_range", "perm_fold_host",
           "perm_plan_complex", "perm_compute_async", "perm_compute_partial", "perm_plan_export",
           "perm_plan_import", "perm_comm_unique_id", "perm_comm_init", "perm_comm_destroy", "perm_probe_fp64_peak"]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libperm.so not built at {LIB_PATH}; run `python -m paper_2501_15126_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i32p = ctypes.POINTER(ctypes.c_int32)
    dp = ctypes.POINTER(ctypes.c_double)
    P = ctypes.c_void_p
    L.perm_plan.argtypes = [ctypes.c_int, ctypes.c_int, i32p, i32p, dp, ctypes.c_int, ctypes.POINTER(P)]
    L.perm_plan_ex.argtypes = [ctypes.c_int, ctypes.c_int, i32p, i32p, dp, ctypes.c_int,
                               ctypes.POINTER(perm_opts), ctypes.POINTER(P)]
    L.perm_plan_complex.argtypes = [ctypes.c_int, ctypes.c_int, i32p, i32p, dp, ctypes.c_int,
                                    ctypes.POINTER(perm_opts), ctypes.POINTER(P)]
    L.perm_compute.restype = ctypes.c_double
    L.perm_compute.argtypes = [P]
    L.perm_compute_ex.argtypes = [P, ctypes.POINTER(perm_result)]
    L.perm_compute_shard.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(perm_result)]
    L.perm_compute_shard_async.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    L.perm_fold.argtypes = [P, ctypes.POINTER(perm_result), ctypes.c_int, ctypes.POINTER(perm_result)]
    L.perm_fold_async.argtypes = [P, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    L.perm_partial_bytes.argtypes = [P]
    L.perm_debug_task_partials.argtypes = [P, ctypes.c_void_p, ctypes.c_uint64,
                                           ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    L.perm_last_timing.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    L.perm_plan_get_info.argtypes = [P, ctypes.POINTER(perm_plan_info)]
    L.perm_plan_source.restype = ctypes.c_char_p
    L.perm_plan_source.argtypes = [P]
    L.perm_plan_cubin.argtypes = [P, ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]
    L.perm_free.restype = None
    L.perm_free.argtypes = [P]
    L.perm_last_error.restype = ctypes.c_char_p
    L.perm_version.restype = ctypes.c_char_p
    L.perm_structural_rank.argtypes = [ctypes.c_int, ctypes.c_int, i32p, i32p, dp]
    L.perm_order.argtypes = [ctypes.c_int, ctypes.c_int, i32p, i32p, dp, ctypes.c_int, i32p, i32p]
    L.perm_partition.argtypes = [ctypes.c_int, i32p, i32p, ctypes.c_double, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    L.perm_alg2_launch_parameters.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                              ctypes.c_int]
    u64p = ctypes.POINTER(ctypes.c_uint64)
    L.perm_shard_range.argtypes = [P, ctypes.c_int, ctypes.c_int, u64p, u64p, u64p, u64p]
    L.perm_fold_host.restype = ctypes.c_double
    L.perm_fold_host.argtypes = [P, dp, ctypes.c_int]
    L.perm_compute_async.argtypes = [P, ctypes.c_void_p]
    L.perm_compute_partial.argtypes = [P, ctypes.c_int, ctypes.c_int, dp]
    L.perm_plan_export.argtypes = [P, ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]
    L.perm_plan_import.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(perm_opts), ctypes.POINTER(P)]
    L.perm_comm_unique_id.argtypes = [ctypes.c_void_p]
    L.perm_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(P)]
    L.perm_comm_destroy.argtypes = [P]
    L.perm_probe_fp64_peak.argtypes = [ctypes.c_int, dp, dp]
    _lib = L
    return L
