"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Each pin is something the paper or mathematics fixes: closed forms, brute
force on tiny inputs, invariants, textbook special cases.  Chosen so that a
dropped term, a wrong sign/index or a transposed operand in any oracle mode
fails at least one test.  CPU only (no GPU marker).
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle
import synth
from conftest import GOLDEN


def golden_closed_forms():
    out = {}
    for line in open(os.path.join(GOLDEN, "closed_forms.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, v = line.split()
        out[k] = int(v)
    return out


def brute_perm(A):
    """Eq. 1 typed out independently with itertools (tiny n only)."""
    n = A.shape[0]
    return sum(math.prod(A[i, s[i]] for i in range(n)) for s in itertools.permutations(range(n)))


def derangements(n):
    d = [1, 0]
    for k in range(2, n + 1):
        d.append((k - 1) * (d[-1] + d[-2]))
    return d[n]


def fib(k):
    a, b = 0, 1
    for _ in range(k):
        a, b = b, a + b
    return a


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def nw_close(A, exact):
    """long-double NW within its own error bound: |v - e| <= 4e-16 |e| (the
    final rounding to double) + 1e-17 * sum|terms| (u = 2^-64 times the n+log
    operation depth, cancellation-aware)."""
    v, sabs = oracle.perm_nw(A)
    return abs(v - exact) <= 4e-16 * abs(exact) + 1e-17 * sabs


# ---- tiny brute force ------------------------------------------------------

def test_2x2_closed_form():
    A = np.array([[2.0, 3.0], [5.0, 7.0]])
    assert oracle.perm_naive(A) == 2 * 7 + 3 * 5
    assert oracle.perm_nw(A)[0] == 2 * 7 + 3 * 5
    assert oracle.perm_ryser_exact(A) == 29
    assert oracle.perm_nw_exact(A) == 29


def test_3x3_written_out():
    A = np.arange(1, 10, dtype=float).reshape(3, 3)
    a = A
    expect = (a[0, 0] * a[1, 1] * a[2, 2] + a[0, 0] * a[1, 2] * a[2, 1] + a[0, 1] * a[1, 0] * a[2, 2]
              + a[0, 1] * a[1, 2] * a[2, 0] + a[0, 2] * a[1, 0] * a[2, 1] + a[0, 2] * a[1, 1] * a[2, 0])
    assert expect == 450
    for f in (oracle.perm_naive, lambda M: oracle.perm_nw(M)[0]):
        assert f(A) == pytest.approx(450, rel=1e-15)
    assert oracle.perm_ryser_exact(A) == 450
    assert oracle.perm_nw_exact(A) == 450
    assert oracle.perm_naive_exact(A) == 450


def test_1x1():
    A = np.array([[3.25]])
    assert oracle.perm_naive(A) == 3.25
    assert oracle.perm_nw(A)[0] == 3.25
    assert oracle.perm_nw_exact(np.array([[-4]])) == -4


@pytest.mark.parametrize("seed", range(6))
def test_random_real_vs_brute(seed):
    rng = np.random.default_rng(seed)
    n = 3 + seed % 4
    A = rng.uniform(-1, 1, (n, n)) * (rng.uniform(size=(n, n)) < 0.7)
    b = brute_perm(A)
    assert abs(oracle.perm_naive(A) - b) <= 1e-13 * abs(b) + 1e-300
    v, sabs = oracle.perm_nw(A)
    assert abs(v - b) <= 1e-15 * max(abs(b), sabs)


# ---- closed forms ----------------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 5, 8, 12, 16, 20])
def test_identity(n):
    I = np.eye(n)
    assert oracle.perm_nw(I)[0] == pytest.approx(1.0, rel=1e-15)
    assert oracle.perm_nw_exact(I) == 1
    if n <= 10:
        assert oracle.perm_naive(I) == 1.0
    if n <= 12:
        assert oracle.perm_ryser_exact(I) == 1
    assert oracle.perm_band(I, 1) == 1.0


@pytest.mark.parametrize("n", [2, 5, 8, 12, 16, 20])
def test_all_ones_factorial(n):
    J = np.ones((n, n))
    assert oracle.perm_nw_exact(J) == math.factorial(n)
    assert rel(oracle.perm_nw(J)[0], math.factorial(n)) < 1e-15
    if n <= 9:
        assert oracle.perm_naive_exact(J) == math.factorial(n)
    if n <= 12:
        assert oracle.perm_ryser_exact(J) == math.factorial(n)
    if n == 20:
        assert oracle.perm_nw_exact(J) == golden_closed_forms()["FACT20"]


@pytest.mark.parametrize("n", [3, 6, 10, 14, 20])
def test_derangements(n):
    A = synth.derangement_matrix(n)
    d = derangements(n)
    assert oracle.perm_nw_exact(A) == d
    assert rel(oracle.perm_nw(A)[0], d) < 1e-14
    if n <= 10:
        assert oracle.perm_naive_exact(A) == d
        assert oracle.perm_ryser_exact(A) == d
    g = golden_closed_forms()
    if n == 10:
        assert d == g["D10"]
    if n == 20:
        assert d == g["D20"]


@pytest.mark.parametrize("n", [1, 2, 3, 10, 20, 44])
def test_tridiagonal_fibonacci(n):
    A = synth.tridiagonal01(n)
    f = fib(n + 1)
    assert oracle.perm_band_exact(A, 1) == f
    assert oracle.perm_band(A, 1) == float(f)
    if n <= 20:
        assert oracle.perm_nw_exact(A) == f
        assert oracle.perm_nw(A)[0] == pytest.approx(f, rel=1e-15)
    if n == 44:
        assert f == golden_closed_forms()["F45"]


def test_triangular_is_diagonal_product():
    rng = np.random.default_rng(3)
    n = 12
    A = np.triu(rng.uniform(0.5, 2.0, (n, n)))
    d = float(np.prod(np.diag(A)))
    assert nw_close(A, d)
    assert nw_close(A.T, d)


def test_zero_row_gives_zero():
    rng = np.random.default_rng(4)
    A = rng.uniform(size=(9, 9))
    A[4, :] = 0
    assert oracle.perm_naive(A) == 0.0
    assert abs(oracle.perm_nw(A)[0]) < 1e-12
    assert oracle.structural_rank(A) == 8


@pytest.mark.parametrize("n,b,seed", [(8, 4, 1), (16, 4, 2), (16, 8, 3), (24, 8, 4)])
def test_block_rank1_closed_form(n, b, seed):
    A, blocks = synth.block_rank1(n, b, seed)
    cf = math.prod(math.factorial(b) * float(np.prod(u)) * float(np.prod(v)) for u, v in blocks)
    assert rel(oracle.perm_nw(A)[0], cf) < 1e-13


def test_block_diagonal_product():
    rng = np.random.default_rng(11)
    B1 = rng.uniform(size=(4, 4))
    B2 = rng.uniform(size=(5, 5))
    A = np.zeros((9, 9))
    A[:4, :4] = B1
    A[4:, 4:] = B2
    assert rel(oracle.perm_nw(A)[0], brute_perm(B1) * brute_perm(B2)) < 1e-13


# ---- cross-mode equalities on random inputs --------------------------------

@pytest.mark.parametrize("seed", range(10))
def test_integer_modes_agree(seed):
    rng = np.random.default_rng(100 + seed)
    n = 2 + seed % 8
    A = rng.integers(-3, 4, (n, n)) * (rng.uniform(size=(n, n)) < 0.6)
    e = oracle.perm_naive_exact(A)
    assert oracle.perm_ryser_exact(A) == e
    assert oracle.perm_nw_exact(A) == e
    assert e == round(brute_perm(A.astype(float))) if n <= 7 else True


@pytest.mark.parametrize("seed", range(8))
def test_er_real_naive_vs_nw(seed):
    n = 5 + seed % 5
    A = synth.erdos_renyi(n, 0.3 + 0.05 * seed, seed)
    assert rel(oracle.perm_nw(A)[0], oracle.perm_naive(A)) < 1e-13


@pytest.mark.parametrize("seed", range(6))
def test_band_dp_vs_naive(seed):
    rng = np.random.default_rng(200 + seed)
    n, w = 7 + seed % 3, 1 + seed % 3
    A = rng.integers(1, 5, (n, n)).astype(float)
    for i in range(n):
        for j in range(n):
            if abs(i - j) > w:
                A[i, j] = 0
    A[rng.uniform(size=(n, n)) < 0.2] = 0
    assert oracle.perm_band_exact(A, w) == oracle.perm_naive_exact(A)
    assert oracle.perm_band(A, w) == pytest.approx(oracle.perm_naive(A), rel=1e-15)


def test_band_brickwork_matches_nw():
    A = synth.givens_brickwork(20, 4, 7)
    w = synth.half_bandwidth(A)
    assert w <= 4
    assert rel(oracle.perm_nw(A)[0], oracle.perm_band(A, w)) < 1e-12


# ---- invariants ------------------------------------------------------------

def test_permutation_and_transpose_invariance():
    A = synth.erdos_renyi(14, 0.3, 5)
    p = oracle.perm_nw(A)[0]
    rng = np.random.default_rng(1)
    P, Q = rng.permutation(14), rng.permutation(14)
    assert rel(oracle.perm_nw(A[np.ix_(P, Q)])[0], p) < 1e-13
    assert rel(oracle.perm_nw(A.T)[0], p) < 1e-13


def test_multilinearity_in_a_row():
    A = synth.erdos_renyi(12, 0.35, 6)
    p = oracle.perm_nw(A)[0]
    B = A.copy()
    B[3] *= -2.5
    assert rel(oracle.perm_nw(B)[0], -2.5 * p) < 1e-13


def test_nw_range_additivity_and_scale():
    A = synth.erdos_renyi(16, 0.3, 9)
    n = 16
    N = 1 << (n - 1)
    total, _ = oracle.nw_range(A, 0, N)
    a, _ = oracle.nw_range(A, 0, 12345)
    b, _ = oracle.nw_range(A, 12345, N)
    assert a + b == pytest.approx(total, rel=1e-12, abs=1e-12 * abs(total))
    assert total * (4 * (n % 2) - 2) == pytest.approx(oracle.perm_naive(A) if n <= 10 else oracle.perm_nw(A)[0])


def test_nw_exact_checksum_divisibility():
    A = synth.erdos_renyi(12, 0.3, 2, binary=True)
    T, zeros = oracle.nw2_range_exact(A, 0, 1 << 11)
    assert T % (1 << 11) == 0
    assert zeros > 0


# ---- structural rank -------------------------------------------------------

def brute_rank(A):
    n = A.shape[0]
    best = 0
    for k in range(n, 0, -1):
        for rows in itertools.combinations(range(n), k):
            for cols in itertools.permutations(range(n), k):
                if all(A[r, c] != 0 for r, c in zip(rows, cols)):
                    return k
    return best


def test_structural_rank_cases():
    assert oracle.structural_rank(np.eye(3)) == 3
    A = np.zeros((3, 3))
    A[:, 0] = 1
    assert oracle.structural_rank(A) == 1
    rng = np.random.default_rng(7)
    for _ in range(6):
        A = (rng.uniform(size=(5, 5)) < 0.3).astype(float)
        assert oracle.structural_rank(A) == brute_rank(A)


# ---- complex permanents --------------------------------------

def brute_perm_c(A):
    n = A.shape[0]
    return sum(math.prod(A[i, s[i]] for i in range(n)) for s in itertools.permutations(range(n)))


def test_complex_2x2_and_diagonal():
    A = np.array([[1 + 2j, 3 - 1j], [0.5j, 2 + 0j]])
    exp = A[0, 0] * A[1, 1] + A[0, 1] * A[1, 0]
    assert abs(oracle.perm_naive_complex(A) - exp) < 1e-15
    assert abs(oracle.perm_nw_complex(A)[0] - exp) < 1e-14
    D = np.diag([1 + 1j, 2 - 0.5j, -1j, 0.25 + 3j, 1.5])
    assert abs(oracle.perm_nw_complex(D)[0] - np.prod(np.diag(D))) < 1e-13


@pytest.mark.parametrize("n", [3, 6, 9])
def test_complex_scaled_ones(n):
    z = 0.7 - 0.4j
    exp = math.factorial(n) * z ** n
    assert abs(oracle.perm_naive_complex(z * np.ones((n, n))) - exp) <= 1e-14 * abs(exp)
    assert abs(oracle.perm_nw_complex(z * np.ones((n, n)))[0] - exp) <= 1e-13 * abs(exp)


@pytest.mark.parametrize("seed", range(5))
def test_complex_naive_vs_brute_and_nw(seed):
    n = 4 + seed % 4
    A = synth.erdos_renyi_complex(n, 0.5, seed)
    b = brute_perm_c(A)
    v, sabs = oracle.perm_nw_complex(A)
    assert abs(oracle.perm_naive_complex(A) - b) <= 1e-14 * max(abs(b), 1e-300) + 1e-300
    assert abs(v - b) <= 1e-15 * sabs
    # conjugation and real-part consistency
    assert abs(oracle.perm_naive_complex(A.conj()) - b.conjugate()) <= 1e-14 * max(abs(b), 1e-300)
    R = np.abs(A)
    assert abs(oracle.perm_nw_complex(R)[0] - oracle.perm_nw(R)[0]) <= 1e-13 * abs(oracle.perm_nw(R)[0])


def test_complex_unitary_brickwork_vs_band_structure():
    U = synth.unitary_brickwork(10, 3, 1)
    assert np.allclose(U.conj().T @ U, np.eye(10))
    assert synth.half_bandwidth(U) <= 3
    v, sabs = oracle.perm_nw_complex(U)
    assert abs(v - oracle.perm_naive_complex(U)) <= 1e-14 * sabs
    rng = np.random.default_rng(3)
    P, Q = rng.permutation(10), rng.permutation(10)
    assert abs(oracle.perm_nw_complex(U[np.ix_(P, Q)])[0] - v) <= 1e-14 * sabs


def test_complex_block_diagonal_product():
    rng = np.random.default_rng(5)
    B1 = rng.normal(size=(3, 3)) + 1j * rng.normal(size=(3, 3))
    B2 = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
    A = np.zeros((7, 7), dtype=complex)
    A[:3, :3] = B1
    A[3:, 3:] = B2
    exp = brute_perm_c(B1) * brute_perm_c(B2)
    v, sabs = oracle.perm_nw_complex(A)
    assert abs(v - exp) <= 1e-14 * sabs


def test_complex_band_dp_vs_naive_and_nw():
    U = synth.unitary_brickwork(12, 3, 2)
    w = synth.half_bandwidth(U)
    b = oracle.perm_band_complex(U, w)
    v, sabs = oracle.perm_nw_complex(U)
    assert abs(b - v) <= 1e-14 * sabs
    assert abs(b - oracle.perm_naive_complex(U)) <= 1e-14 * sabs


# ---- round 2: pins for the remaining oracle surfaces ---------------------------

def test_nw2_zero_count_by_brute_force():
    """nw2_range_exact's second output = number of Gray states g in the range
    with some x_i(Gray_g) = 0 (the zero-tracking quantity of Sec. VI-B, P:589,
    P:684).  Brute force over subsets S of columns 0..n-2, typed out from the
    doubled form 2x_i(S) = 2a_{i,n-1} - r_i + 2 sum_{j in S} a_ij."""
    for seed in (2, 3, 5):
        A = synth.erdos_renyi(10, 0.3, seed, binary=True).astype(np.int64)
        n = 10
        r = A.sum(axis=1)
        zeros_all = 0
        for mask in range(1 << (n - 1)):
            x2 = 2 * A[:, n - 1] - r + 2 * sum(A[:, j] for j in range(n - 1) if mask >> j & 1)
            zeros_all += bool((x2 == 0).any())
        T, z = oracle.nw2_range_exact(A, 0, 1 << (n - 1))
        assert z == zeros_all                       # the Gray walk visits every subset once
        # and over a sub-range: count the Gray codes g ^ (g >> 1) it visits
        lo, hi = 37, 300
        zr = 0
        for g in range(lo, hi):
            mask = g ^ (g >> 1)
            x2 = 2 * A[:, n - 1] - r + 2 * sum(A[:, j] for j in range(n - 1) if mask >> j & 1)
            zr += bool((x2 == 0).any())
        assert oracle.nw2_range_exact(A, lo, hi)[1] == zr


def test_nw_range_complex_additivity_and_scale():
    rng = np.random.default_rng(11)
    n = 8
    A = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) * (rng.uniform(size=(n, n)) < 0.6)
    A += np.eye(n)
    N = 1 << (n - 1)
    total, _ = oracle.nw_range_complex(A, 0, N)
    a, _ = oracle.nw_range_complex(A, 0, 41)
    b, _ = oracle.nw_range_complex(A, 41, N)
    assert abs((a + b) - total) <= 1e-12 * abs(total)
    bp = brute_perm_c(A)
    assert abs(total * (4 * (n % 2) - 2) - bp) <= 1e-12 * abs(bp)


def test_nw_range_f64_within_double_error_bound():
    """The double-precision sweep (CPU-baseline leg) agrees with the long-double
    oracle within u_double * (n + chunk depth) * sum|terms|, and is exact where
    every x and product is a small dyadic rational (0/1 inputs: half-integers)."""
    for seed in range(3):
        A = synth.erdos_renyi(18, 0.3, seed)
        N = 1 << 17
        s_ld, a_ld = oracle.nw_range(A, 0, N)
        s_d, a_d = oracle.nw_range_f64(A, 0, N)
        assert abs(s_d - s_ld) <= 2.0 ** -53 * 64 * a_ld
        assert abs(a_d - a_ld) <= 1e-12 * a_ld
    B = synth.erdos_renyi(16, 0.3, 4, binary=True)
    T, _ = oracle.nw2_range_exact(B, 0, 1 << 15)
    s_d, _ = oracle.nw_range_f64(B, 0, 1 << 15)
    assert s_d * 2 ** 16 == T          # x = x'/2 exact, products of <= 16 half-integers exact
