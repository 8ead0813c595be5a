"""oracle/planner.py -- plain-Python ORACLE for the host-planner rows of the path.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import this module.  It shares no code with the product
(paper_2501_15126_b200/), which implements the same algorithms in C++.

Each function follows the paper passage it cites, in the paper's order and
notation (P:n = /root/reference/PAPER.md line n).  Pure-Python loops: meant for
small inputs and for exact (integer) parity against the product planner.
"""
from __future__ import annotations

from fractions import Fraction


# --- Gray codes (Alg. 1 line 9; Sec. IV) -------------------

def gray(g: int) -> int:
    """g-th reflected Gray code, Gray_g = g XOR (g >> 1)."""
    return g ^ (g >> 1)


def changed_bit(g: int) -> tuple[int, int]:
    """(j, s) of Alg. 1 lines 9-10 computed literally from the codes:
    j = log2(Gray_g XOR Gray_{g-1}), s = 2*Gray_g[j] - 1."""
    d = gray(g) ^ gray(g - 1)
    j = d.bit_length() - 1
    s = 2 * ((gray(g) >> j) & 1) - 1
    return j, s


def scbs_entry(i: int) -> tuple[int, int]:
    """Theorem 1: entry i >= 1 of SCBS has column j with 2^j the
    largest power of two dividing i; sign + iff (i - 2^j)/2^(j+1) is even."""
    if i < 1:
        raise ValueError("SCBS positions start at 1")
    j = 0
    while i % (2 ** (j + 1)) == 0:
        j += 1
    s = +1 if ((i - 2 ** j) // 2 ** (j + 1)) % 2 == 0 else -1
    return j, s


def scbs_recursive(k: int) -> list[tuple[int, int]]:
    """SCBS(k) = [SCBS(k-1), +(k-1), -SCBS(k-1)^R]."""
    if k < 1:
        raise ValueError("k >= 1")
    if k == 1:
        return [(0, +1)]
    prev = scbs_recursive(k - 1)
    return prev + [(k - 1, +1)] + [(j, -s) for (j, s) in reversed(prev)]


def appearance_count(n: int, j: int) -> int:
    """Lemma 2: column j appears 2^(n-j-2) times in SCBS(n-1)."""
    if not 0 <= j < n - 1:
        raise ValueError("0 <= j < n-1")
    return 2 ** (n - j - 2)


def update_probability(n: int, cols) -> tuple[Fraction, Fraction]:
    """Sec. V: probability that a row touched by `cols` is modified in
    an iteration: exact sum 2^(n-j-2)/(2^(n-1)-1) and the paper's 2^-(j+1)."""
    exact = sum((Fraction(2 ** (n - j - 2), 2 ** (n - 1) - 1) for j in cols), Fraction(0))
    approx = sum((Fraction(1, 2 ** (j + 1)) for j in cols), Fraction(0))
    return exact, approx


# --- Alg. 2 GenerateLaunchParameters -----------------------------

def generate_launch_parameters(tau: int, n: int) -> list[tuple[int, int, int]]:
    """Alg. 2 verbatim: list of (start, Delta, end)."""
    K = []
    start = 1
    end = 2 ** (n - 1)
    while end - start > 0:
        delta = 1024
        while delta * tau <= end - start:
            delta *= 2
        delta //= 2
        if delta == 512:
            K.append((start, 1024, end))
            break
        K.append((start, delta, end))
        start = start + tau * delta
    return K


def chunk_of(spec: tuple[int, int, int], t: int, n: int):
    """Chunk of thread t in launch `spec` (Sec. II-A; Alg. 2 note P:341):
    (g_start, g_end) inclusive, or None when past the last iteration."""
    start, delta, _end = spec
    gs = start + t * delta
    last = 2 ** (n - 1) - 1
    if gs > last:
        return None
    return gs, min(gs + delta - 1, last)


def divergence_of_schedule(n: int, chunk: int, tau: int, warp: int) -> list[int]:
    """Sec. IV table: number of distinct signed kernels per local
    iteration across a warp of `warp` threads, chunks g_start = t*chunk + 1."""
    last = 2 ** (n - 1) - 1
    out = []
    for w0 in range(0, tau, warp):
        for ell in range(chunk):
            kinds = set()
            for t in range(w0, min(w0 + warp, tau)):
                i = t * chunk + 1 + ell
                if i <= last:
                    kinds.add(scbs_entry(i))
            if kinds:
                out.append(len(kinds))
    return out


# --- Alg. 3 PermanentOrdering ------------------------------------

def permanent_ordering(n: int, cptrs, rids, rptrs, cids):
    """Alg. 3 verbatim.  Readings (DESIGN R11): argmin ties -> lowest column
    index; rows of `col` visited in CSC order; rows never reached are appended
    in original order.  Returns (rowPerm, colPerm): new position -> original."""
    INF = float("inf")
    cdeg = [cptrs[j + 1] - cptrs[j] for j in range(n)]        # lines 1-3
    rmark = [False] * n                                         # lines 4-6
    rowPerm, colPerm = [], []
    for _cidx in range(n):                                      # line 8
        col = min(range(n), key=lambda j: (cdeg[j], j))        # line 10
        colPerm.append(col)                                     # line 11
        cdeg[col] = INF                                         # line 12
        for p in range(cptrs[col], cptrs[col + 1]):             # line 13
            row = rids[p]
            if not rmark[row]:                                  # line 15
                rmark[row] = True                               # line 16
                rowPerm.append(row)                             # line 17
                for q in range(rptrs[row], rptrs[row + 1]):     # line 20
                    cdeg[cids[q]] -= 1                          # line 21
    for r in range(n):
        if not rmark[r]:
            rowPerm.append(r)
    return rowPerm, colPerm


def degree_sort_ascending(n: int, cptrs):
    """Sec. VI-B: columns by nonzero count ascending, ties by index."""
    return sorted(range(n), key=lambda j: (cptrs[j + 1] - cptrs[j], j))


# --- Alg. 4 Partitioning -----------------------------------------

def calculate_no_threads(nregisters: int, sms: int = 148, regs_per_sm: int = 65536,
                         max_threads_per_sm: int = 2048, max_regs: int = 255,
                         overhead: int = 32, warp: int = 32) -> int:
    """CalculateNoThreads (undefined in the paper): register-limited
    resident threads.  Model: regs per thread = nregisters + overhead, threads
    per SM rounded down to whole warps, capped by the thread limit."""
    per = nregisters + overhead
    if per > max_regs:
        return 0
    t = (regs_per_sm // per) // warp * warp
    return sms * min(max_threads_per_sm, t)


def partitioning(n: int, cptrs, rids, gr_ratio: float = 16.0, tau_fn=calculate_no_threads):
    """Alg. 4 verbatim on an ORDERED matrix's CSC. Returns (k, c)."""
    k = 0
    c = 0
    best = 0.0
    nrows = 0
    for j in range(n):                                                   # line 5
        if cptrs[j + 1] > cptrs[j]:
            nrows = max(nrows, max(rids[cptrs[j]:cptrs[j + 1]]) + 1)     # line 7
        nreg = nrows * 2                                                 # line 8
        reg_cost = nreg * (1 - 2.0 ** (-(j + 1)))                        # line 9
        glob_cost = (n - nrows) * 2.0 ** (-(j + 1)) * gr_ratio           # line 10
        tau = tau_fn(nreg)                                               # line 12
        denom = reg_cost + glob_cost
        score = tau / denom if denom > 0 else 0.0                        # line 13
        if score > best or nrows == k:                                   # line 14
            best = score
            k = nrows
            c = j + 1
    return k, c
