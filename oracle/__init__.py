"""oracle -- plain, slow, obviously-correct CPU oracle for the sparse permanent.

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import, call, link or execute anything
under oracle/.  The product (paper_2501_15126_b200/) never imports it and the
two share no code: the oracle takes dense row-major matrices and has its own
C++ source (oracle.cpp) and its own Python planner (planner.py).

Functions (each cites its passage; P:n = /root/reference/PAPER.md line n):
  perm_naive        Eq. 1, long double or exact int128
  perm_ryser_exact  Eq. 2, exact int128, integer inputs
  perm_nw           Alg. 1 + Sec. II-A chunking, long double
  nw_range          unscaled Alg. 1 partial sum over a Gray range (long double)
  nw_range_f64      the same in IEEE double (CPU-baseline leg)
  nw2_range_exact   Alg. 1 in exact doubled integers (integer inputs)
  perm_band         band DP (exact textbook evaluation of Eq. 1 for banded A)
  structural_rank   maximum bipartite matching
  nw_range_complex, perm_naive_complex, perm_band_complex, perm_nw_complex
                    the same over C (complex long double)
oracle/planner.py restates Sec. IV (Theorem 1, SCBS, Lemma 1/2), Alg. 2, Alg. 3,
the degree sort and Alg. 4, and nothing else.
Every function is pinned against something other than itself in
tests/test_oracle.py / tests/test_planner_oracle.py (closed forms, brute force,
printed examples, invariants); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -fopenmp).  No fast-math: long double
    rounding must be IEEE/x87-exact."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared", _SRC, "-o", _LIB + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            u64p = ctypes.POINTER(ctypes.c_uint64)
            ldp = ctypes.POINTER(ctypes.c_longdouble)
            dp = ctypes.POINTER(ctypes.c_double)
            i64p = ctypes.POINTER(ctypes.c_int64)
            L.oracle_perm_naive_ld.restype = ctypes.c_longdouble
            L.oracle_perm_naive_ld.argtypes = [ctypes.c_int, dp]
            L.oracle_perm_naive_i128.argtypes = [ctypes.c_int, i64p, u64p, u64p]
            L.oracle_perm_ryser_i128.argtypes = [ctypes.c_int, i64p, ctypes.c_int, u64p, u64p]
            L.oracle_nw_range_ld.argtypes = [ctypes.c_int, dp, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_int, ldp, ldp]
            L.oracle_nw_range_d.argtypes = [ctypes.c_int, dp, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_int, dp, dp]
            L.oracle_perm_nw_ld.restype = ctypes.c_longdouble
            L.oracle_perm_nw_ld.argtypes = [ctypes.c_int, dp, ctypes.c_int, ldp]
            L.oracle_nw2_range_i128.argtypes = [ctypes.c_int, i64p, ctypes.c_uint64, ctypes.c_uint64,
                                                ctypes.c_int, u64p, u64p, u64p]
            L.oracle_perm_band_ld.restype = ctypes.c_longdouble
            L.oracle_perm_band_ld.argtypes = [ctypes.c_int, dp, ctypes.c_int]
            L.oracle_perm_band_i128.argtypes = [ctypes.c_int, i64p, ctypes.c_int, u64p, u64p]
            L.oracle_structural_rank.restype = ctypes.c_int
            L.oracle_structural_rank.argtypes = [ctypes.c_int, dp]
            L.oracle_max_threads.restype = ctypes.c_int
            L.oracle_perm_naive_c.argtypes = [ctypes.c_int, dp, ldp, ldp]
            L.oracle_perm_band_c.argtypes = [ctypes.c_int, dp, ctypes.c_int, ldp, ldp]
            L.oracle_nw_range_c.argtypes = [ctypes.c_int, dp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                            ldp, ldp, ldp]
            _lib = L
    return _lib


def _dense_f64(A) -> np.ndarray:
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("square matrix required")
    return A


def _dense_i64(A) -> np.ndarray:
    Af = np.asarray(A)
    Ai = np.ascontiguousarray(np.asarray(Af, dtype=np.int64))
    if not np.array_equal(Ai, Af):
        raise ValueError("integer matrix required")
    if Ai.ndim != 2 or Ai.shape[0] != Ai.shape[1]:
        raise ValueError("square matrix required")
    return Ai


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _signed128(lo: int, hi: int) -> int:
    v = (hi << 64) | lo
    return v - (1 << 128) if v >> 127 else v


def max_threads() -> int:
    return _load().oracle_max_threads()


def perm_naive(A) -> float:
    """Eq. 1 in long double (returned as Python float of the long double)."""
    A = _dense_f64(A)
    return float(_load().oracle_perm_naive_ld(A.shape[0], _dp(A)))


def perm_naive_exact(A) -> int:
    """Eq. 1 in exact integers."""
    A = _dense_i64(A)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    _load().oracle_perm_naive_i128(A.shape[0], _ip(A), ctypes.byref(lo), ctypes.byref(hi))
    return _signed128(lo.value, hi.value)


def perm_ryser_exact(A, threads: int = 0) -> int:
    """Eq. 2 (Ryser) in exact integers (mod 2^128, signed)."""
    A = _dense_i64(A)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    _load().oracle_perm_ryser_i128(A.shape[0], _ip(A), threads, ctypes.byref(lo), ctypes.byref(hi))
    return _signed128(lo.value, hi.value)


def nw_range(A, g_begin: int, g_end: int, threads: int = 0):
    """Unscaled Alg. 1 partial sum over g in [g_begin, g_end):
    sum (-1)^g prod_i x_i(Gray_g) in long double.  Returns (sum, sum|terms|)
    as Python floats (rounded from long double)."""
    A = _dense_f64(A)
    s, a = ctypes.c_longdouble(), ctypes.c_longdouble()
    _load().oracle_nw_range_ld(A.shape[0], _dp(A), g_begin, g_end, threads,
                               ctypes.byref(s), ctypes.byref(a))
    return float(s.value), float(a.value)


def nw_range_f64(A, g_begin: int, g_end: int, threads: int = 0):
    """nw_range in IEEE double (same chunking and fold): the FP64 analogue of
    the paper's CPU-SparsePerman, used as a CPU baseline leg."""
    A = _dense_f64(A)
    s, a = ctypes.c_double(), ctypes.c_double()
    _load().oracle_nw_range_d(A.shape[0], _dp(A), g_begin, g_end, threads, ctypes.byref(s), ctypes.byref(a))
    return s.value, a.value


def perm_nw(A, threads: int = 0):
    """perm(A) by Alg. 1 (+ Sec. II-A chunking) in long double.
    Returns (perm, sum|terms|); kappa = sum|terms| / |perm|."""
    A = _dense_f64(A)
    a = ctypes.c_longdouble()
    v = _load().oracle_perm_nw_ld(A.shape[0], _dp(A), threads, ctypes.byref(a))
    return float(v), float(a.value)


def nw2_range_exact(A, g_begin: int, g_end: int, threads: int = 0):
    """Alg. 1 in exact doubled integers over [g_begin, g_end): returns
    (T' signed int (mod 2^128), number of terms with some x_i = 0)."""
    A = _dense_i64(A)
    lo, hi, z = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _load().oracle_nw2_range_i128(A.shape[0], _ip(A), g_begin, g_end, threads,
                                  ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(z))
    return _signed128(lo.value, hi.value), z.value


def perm_nw_exact(A, threads: int = 0) -> int:
    """perm(A) = (-1)^(n-1) T' / 2^(n-1) in exact integers (integer A)."""
    A = _dense_i64(A)
    n = A.shape[0]
    if n == 1:
        return int(A[0, 0])
    T, _ = nw2_range_exact(A, 0, 1 << (n - 1), threads)
    q, r = divmod(T, 1 << (n - 1))
    if r != 0:
        raise ArithmeticError("T' not divisible by 2^(n-1): overflow of the 128-bit range")
    return q if (n - 1) % 2 == 0 else -q


def perm_band(A, w: int) -> float:
    A = _dense_f64(A)
    return float(_load().oracle_perm_band_ld(A.shape[0], _dp(A), w))


def perm_band_exact(A, w: int) -> int:
    A = _dense_i64(A)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    _load().oracle_perm_band_i128(A.shape[0], _ip(A), w, ctypes.byref(lo), ctypes.byref(hi))
    return _signed128(lo.value, hi.value)


def _dense_c(A) -> np.ndarray:
    A = np.asarray(A, dtype=np.complex128)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("square matrix required")
    return np.ascontiguousarray(A).view(np.float64)   # interleaved (re, im)


def perm_naive_complex(A) -> complex:
    """Eq. 1 over C in complex long double."""
    n = np.asarray(A).shape[0]
    Ai = _dense_c(A)
    re, im = ctypes.c_longdouble(), ctypes.c_longdouble()
    _load().oracle_perm_naive_c(n, _dp(Ai), ctypes.byref(re), ctypes.byref(im))
    return complex(float(re.value), float(im.value))


def perm_band_complex(A, w: int) -> complex:
    """Band DP of Eq. 1 over C (a_ij = 0 for |i - j| > w)."""
    n = np.asarray(A).shape[0]
    Ai = _dense_c(A)
    re, im = ctypes.c_longdouble(), ctypes.c_longdouble()
    _load().oracle_perm_band_c(n, _dp(Ai), w, ctypes.byref(re), ctypes.byref(im))
    return complex(float(re.value), float(im.value))


def nw_range_complex(A, g_begin: int, g_end: int, threads: int = 0):
    """Unscaled complex Alg. 1 partial over [g_begin, g_end): (sum, sum|terms|)."""
    n = np.asarray(A).shape[0]
    Ai = _dense_c(A)
    re, im, sa = ctypes.c_longdouble(), ctypes.c_longdouble(), ctypes.c_longdouble()
    _load().oracle_nw_range_c(n, _dp(Ai), g_begin, g_end, threads, ctypes.byref(re), ctypes.byref(im),
                              ctypes.byref(sa))
    return complex(float(re.value), float(im.value)), float(sa.value)


def perm_nw_complex(A, threads: int = 0):
    """perm(A) over C by Alg. 1 (+ Sec. II-A chunking), complex long double;
    returns (perm, 2 * sum|terms|)."""
    n = np.asarray(A).shape[0]
    if n == 1:
        v = complex(np.asarray(A)[0, 0])
        return v, abs(v)
    s, a = nw_range_complex(A, 0, 1 << (n - 1), threads)
    f = 4 * (n % 2) - 2   # line 23
    return s * f, 2 * a


def structural_rank(A) -> int:
    A = _dense_f64(A)
    return int(_load().oracle_structural_rank(A.shape[0], _dp(A)))
