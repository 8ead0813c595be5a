"""synth -- seeded synthetic inputs shared by the oracle tests, the GPU parity
tests and bench.py.  Holds NONE of the method's arithmetic: it only draws
matrices and converts between dense / CCS / CRS / Matrix Market layouts.

Input recipe (paper P:655-657):
  * SplitMix64(seed) stream; u = (z >> 11) * 2^-53 in [0, 1).
  * Erdos-Renyi(n, p): row-major cells, cell nonzero iff u < p; its value is
    1 - u' in (0, 1] (never an explicit zero).  Draws whose structural rank is
    below n are rejected and the stream continues.
  * 0/1 ER: same pattern draw, all values 1.0.
  * Band (low-depth boson sampling): real orthogonal brickwork of depth
    D: alternating even/odd layers of Givens rotations on neighbouring modes
    with angles 2*pi*u; half-width <= D.  Variant: same pattern, U(0,1] values.
  * Block-diagonal rank-1 (closed-form pin): b x b blocks u v^T with u, v in
    (0,1]^b, then random row and column permutations.
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        """u in [0, 1) with 53 random bits."""
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def unit_open0(self) -> float:
        """1 - u in (0, 1]."""
        return 1.0 - self.uniform()

    def below(self, m: int) -> int:
        return self.next_u64() % m

    def permutation(self, n: int) -> list[int]:
        p = list(range(n))
        for i in range(n - 1, 0, -1):          # Fisher-Yates
            k = self.below(i + 1)
            p[i], p[k] = p[k], p[i]
        return p


def _has_perfect_matching(A: np.ndarray) -> bool:
    """Rejection test of the generator: a perfect matching of the
    nonzero pattern exists (augmenting paths)."""
    n = A.shape[0]
    adj = [np.nonzero(A[i])[0].tolist() for i in range(n)]
    mcol = [-1] * n

    def aug(i, seen):
        for j in adj[i]:
            if not seen[j]:
                seen[j] = True
                if mcol[j] < 0 or aug(mcol[j], seen):
                    mcol[j] = i
                    return True
        return False

    return all(aug(i, [False] * n) for i in range(n))


def erdos_renyi(n: int, p: float, seed: int, binary: bool = False, max_attempts: int = 1000) -> np.ndarray:
    rng = SplitMix64(seed)
    for _ in range(max_attempts):
        A = np.zeros((n, n), dtype=np.float64)
        for i in range(n):
            for j in range(n):
                if rng.uniform() < p:
                    v = rng.unit_open0()
                    A[i, j] = 1.0 if binary else v
        if _has_perfect_matching(A):
            return A
    raise RuntimeError(f"no structurally nonsingular ER({n},{p}) draw in {max_attempts} attempts")


def givens_brickwork(n: int, depth: int, seed: int) -> np.ndarray:
    """Real orthogonal n x n matrix built from `depth` brickwork layers."""
    rng = SplitMix64(seed)
    U = np.eye(n)
    for layer in range(depth):
        L = np.eye(n)
        for a in range(layer % 2, n - 1, 2):
            th = 2.0 * math.pi * rng.uniform()
            c, s = math.cos(th), math.sin(th)
            L[a, a], L[a, a + 1], L[a + 1, a], L[a + 1, a + 1] = c, -s, s, c
        U = L @ U
    U[np.abs(U) < 1e-300] = 0.0
    return U


def band_positive(n: int, depth: int, seed: int) -> np.ndarray:
    """Same pattern as givens_brickwork(n, depth, seed), values U(0,1]."""
    pat = givens_brickwork(n, depth, seed) != 0
    rng = SplitMix64(seed ^ 0x5DEECE66D)
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if pat[i, j]:
                A[i, j] = rng.unit_open0()
    return A


def erdos_renyi_complex(n: int, p: float, seed: int, max_attempts: int = 1000) -> np.ndarray:
    """ER pattern as erdos_renyi; value r e^{i theta}, r in (0,1], theta = 2 pi u."""
    rng = SplitMix64(seed ^ 0xC0FFEE)
    for _ in range(max_attempts):
        A = np.zeros((n, n), dtype=np.complex128)
        for i in range(n):
            for j in range(n):
                if rng.uniform() < p:
                    r = rng.unit_open0()
                    th = 2.0 * math.pi * rng.uniform()
                    A[i, j] = r * complex(math.cos(th), math.sin(th))
        if _has_perfect_matching(A != 0):
            return A
    raise RuntimeError("no structurally nonsingular complex ER draw")


def unitary_brickwork(n: int, depth: int, seed: int) -> np.ndarray:
    """Complex unitary of `depth` brickwork layers of beam splitters
    [[e^{i phi} cos t, -sin t], [e^{i phi} sin t, cos t]] on neighbouring modes
    (low-depth boson sampling interferometer); half-width <= depth."""
    rng = SplitMix64(seed ^ 0xB05)
    U = np.eye(n, dtype=np.complex128)
    for layer in range(depth):
        L = np.eye(n, dtype=np.complex128)
        for a in range(layer % 2, n - 1, 2):
            t = 2.0 * math.pi * rng.uniform()
            ph = 2.0 * math.pi * rng.uniform()
            e = complex(math.cos(ph), math.sin(ph))
            L[a, a], L[a, a + 1] = e * math.cos(t), -math.sin(t)
            L[a + 1, a], L[a + 1, a + 1] = e * math.sin(t), math.cos(t)
        U = L @ U
    U[np.abs(U) < 1e-300] = 0.0
    return U


def half_bandwidth(A: np.ndarray) -> int:
    ii, jj = np.nonzero(A)
    return int(np.max(np.abs(ii - jj))) if ii.size else 0


def block_rank1(n: int, b: int, seed: int):
    """Block-diagonal rank-1 matrix with random row/column permutations.
    Returns (A, blocks) with blocks = [(u, v), ...] for the closed form."""
    if n % b:
        raise ValueError("b must divide n")
    rng = SplitMix64(seed)
    D = np.zeros((n, n))
    blocks = []
    for k in range(n // b):
        u = np.array([rng.unit_open0() for _ in range(b)])
        v = np.array([rng.unit_open0() for _ in range(b)])
        D[k * b:(k + 1) * b, k * b:(k + 1) * b] = np.outer(u, v)
        blocks.append((u, v))
    P = rng.permutation(n)
    Q = rng.permutation(n)
    return D[np.ix_(P, Q)], blocks


def block_diagonal(n: int, b: int, seed: int):
    """Block-diagonal matrix of dense b x b blocks with U(0,1] entries, then
    random row and column permutations (closed-form pin: perm = product of the
    block permanents; density b/n).  Returns (A, [block matrices])."""
    if n % b:
        raise ValueError("b must divide n")
    rng = SplitMix64(seed ^ 0xB10C)
    D = np.zeros((n, n))
    blocks = []
    for k in range(n // b):
        blk = np.array([[rng.unit_open0() for _ in range(b)] for _ in range(b)])
        D[k * b:(k + 1) * b, k * b:(k + 1) * b] = blk
        blocks.append(blk)
    P = rng.permutation(n)
    Q = rng.permutation(n)
    return D[np.ix_(P, Q)], blocks


def ones(n):
    return np.ones((n, n))


def identity(n):
    return np.eye(n)


def derangement_matrix(n):
    return np.ones((n, n)) - np.eye(n)


def tridiagonal01(n):
    A = np.zeros((n, n))
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                A[i, j] = 1.0
    return A


# ---- layouts ---------------------------------------------------------------

def to_ccs(A: np.ndarray):
    """Dense -> CCS (column pointers, row ids ascending, values) as int32/f64."""
    n = A.shape[0]
    ptr = [0]
    idx, val = [], []
    for j in range(n):
        rows = np.nonzero(A[:, j])[0]
        idx.extend(rows.tolist())
        val.extend(A[rows, j].tolist())
        ptr.append(len(idx))
    vdt = np.complex128 if np.iscomplexobj(A) else np.float64
    return (np.array(ptr, dtype=np.int32), np.array(idx, dtype=np.int32), np.array(val, dtype=vdt))


def to_crs(A: np.ndarray):
    """Dense -> CRS (row pointers, column ids ascending, values)."""
    ptr, idx, val = to_ccs(np.ascontiguousarray(A.T))
    return ptr, idx, val


def write_mtx(path: str, A: np.ndarray) -> None:
    """Matrix Market coordinate real general, 1-based, 17 significant digits."""
    n = A.shape[0]
    ii, jj = np.nonzero(A)
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{n} {n} {ii.size}\n")
        for i, j in zip(ii.tolist(), jj.tolist()):
            f.write(f"{i + 1} {j + 1} {A[i, j]:.17g}\n")


def read_mtx(path: str) -> np.ndarray:
    with open(path) as f:
        header = f.readline().lower().split()
        if len(header) < 5 or header[1] != "matrix" or header[2] != "coordinate":
            raise ValueError("only coordinate Matrix Market files are supported")
        field, sym = header[3], header[4]
        if field == "pattern":
            raise ValueError("pattern-only matrices carry no values")
        line = f.readline()
        while line.startswith("%"):
            line = f.readline()
        m, n, nnz = (int(t) for t in line.split())
        if m != n:
            raise ValueError("square matrix required")
        A = np.zeros((n, n))
        for _ in range(nnz):
            t = f.readline().split()
            i, j, v = int(t[0]) - 1, int(t[1]) - 1, float(t[2])
            A[i, j] = v
            if sym == "symmetric" and i != j:
                A[j, i] = v
    return A
