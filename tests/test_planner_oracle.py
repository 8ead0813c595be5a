"""Pins for the planner oracle (oracle/planner.py) against the paper's printed
examples and exhaustive mathematics.  CPU only."""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import planner as P
import synth
from conftest import GOLDEN


def parse_signed(tok):
    return int(tok[1:]), (+1 if tok[0] == "+" else -1)


def read_golden(name):
    return [l for l in open(os.path.join(GOLDEN, name)) if l.strip() and not l.startswith("#")]


def test_scbs_printed_sequences():
    for line in read_golden("scbs.txt"):
        k, seq = line.split(":")
        expect = [parse_signed(t) for t in seq.split()]
        assert P.scbs_recursive(int(k)) == expect
        assert [P.scbs_entry(i) for i in range(1, 2 ** int(k))] == expect


def test_cbs_5x5():
    expect = [int(t) for t in read_golden("cbs5.txt")[0].split()]
    assert [P.changed_bit(g)[0] for g in range(1, 16)] == expect


def test_theorem1_exhaustive():
    for k in range(1, 15):
        rec = P.scbs_recursive(k)
        for i, e in enumerate(rec, start=1):
            assert P.scbs_entry(i) == e


def test_alg1_lines_9_10_match_theorem1():
    for g in range(1, 1 << 14):
        assert P.changed_bit(g) == P.scbs_entry(g)


def test_lemma2_counts():
    for k in range(1, 13):
        n = k + 1
        seq = P.scbs_recursive(k)
        for j in range(k):
            assert sum(1 for (c, _) in seq if c == j) == P.appearance_count(n, j)
        assert sum(P.appearance_count(n, j) for j in range(k)) == 2 ** k - 1
        # signs of each column's appearances alternate, starting with +
        for j in range(k):
            signs = [s for (c, s) in seq if c == j]
            assert signs == [(-1) ** t for t in range(len(signs))]


def test_update_probabilities_printed():
    # x[2] is touched by columns {0,3,4}: 19/32; x[4] by {1,2}: 3/8
    _, a = P.update_probability(6, [0, 3, 4])
    assert a == Fraction(19, 32)
    _, b = P.update_probability(6, [1, 2])
    assert b == Fraction(3, 8)
    assert P.update_probability(6, [])[0] == 0


def test_divergence_table():
    expect = [int(t) for t in read_golden("divergence5.txt")[0].split()]
    assert P.divergence_of_schedule(5, 3, 5, 32) == expect


def test_lemma1_power_of_two_chunks():
    # with chunk 2^kc and g_start = t*2^kc + 1 (Alg. 2 style), divergence only
    # at local iterations 2^(kc-1)-1 and 2^kc-1 (0-based ell)
    n = 14
    for kc in range(2, 8):
        ch = 2 ** kc
        tau = 64
        counts = P.divergence_of_schedule(n, ch, tau, 32)
        per_warp = [counts[w * ch:(w + 1) * ch] for w in range(tau // 32)]
        for cw in per_warp:
            bad = [ell for ell, c in enumerate(cw) if c > 1]
            assert set(bad) <= {2 ** (kc - 1) - 1, 2 ** kc - 1}
            assert len(bad) <= 2


def test_alg2_trace_and_cover():
    assert P.generate_launch_parameters(4, 16) == [
        (1, 4096, 32768), (16385, 2048, 32768), (24577, 1024, 32768), (28673, 1024, 32768)]
    assert P.generate_launch_parameters(2048, 12) == [(1, 1024, 2048)]
    for tau in (4, 32, 1024):
        for n in (12, 16, 22):
            plan = P.generate_launch_parameters(tau, n)
            last = 2 ** (n - 1) - 1
            covered = 0
            prev_end = 0
            for spec in plan:
                assert spec[1] >= 1024 and spec[1] & (spec[1] - 1) == 0
                for t in range(tau):
                    c = P.chunk_of(spec, t, n)
                    if c is None:
                        continue
                    assert c[0] == prev_end + 1
                    prev_end = c[1]
                    covered += c[1] - c[0] + 1
            assert covered == last and prev_end == last


def csr_csc(A):
    cp, ri, _ = synth.to_ccs(A)
    rp, ci, _ = synth.to_crs(A)
    return cp, ri, rp, ci


def test_alg3_basic_properties():
    n = 10
    A = np.eye(n)
    cp, ri, rp, ci = csr_csc(A)
    rp_, cp_ = P.permanent_ordering(n, cp, ri, rp, ci)
    assert rp_ == list(range(n)) and cp_ == list(range(n))
    # a column with a single nonzero is chosen first
    A = synth.erdos_renyi(12, 0.5, 3)
    A[:, 7] = 0
    A[5, 7] = 0.5
    cp, ri, rp, ci = csr_csc(A)
    rowp, colp = P.permanent_ordering(12, cp, ri, rp, ci)
    assert colp[0] == 7 and rowp[0] == 5
    assert sorted(rowp) == list(range(12)) and sorted(colp) == list(range(12))
    B = A[np.ix_(rowp, colp)]
    assert oracle.perm_nw(B)[0] == pytest.approx(oracle.perm_nw(A)[0], rel=1e-12)


def test_alg4_fig3b_fixture():
    lines = read_golden("fig3b_ordered.txt")
    n = int(lines[0])
    A = np.zeros((n, n))
    for l in lines[1:]:
        r, c, v = l.split()
        A[int(r), int(c)] = float(v)
    # Listing 4: ordered column 3 carries the Listing 2 values
    col0 = {int(l.split()[0]): float(l.split()[1]) for l in read_golden("listing2_col0.txt")}
    assert sorted(A[:, 3][A[:, 3] != 0].tolist()) == sorted(col0.values())
    cp, ri, _, _ = csr_csc(A)
    a100 = lambda r: P.calculate_no_threads(r, sms=108)
    assert P.partitioning(n, cp, ri, 16.0, a100) == (4, 3)


def test_calculate_no_threads_calibration():
    # SPEC-derived calibration: 96 regs under the A100 model -> 55296
    assert P.calculate_no_threads(96, sms=108) == 55296
    assert P.calculate_no_threads(0, sms=108) == 108 * 2048
    assert P.calculate_no_threads(240) == 0


@pytest.mark.parametrize("p", [0.1, 0.2, 0.3])
def test_alg4_region_invariant_and_ordering_trend(p):
    n = 40
    ks_ord, ks_raw = [], []
    for seed in range(8):
        A = synth.erdos_renyi(n, p, seed)
        cp, ri, rp, ci = csr_csc(A)
        k_raw, _ = P.partitioning(n, cp, ri)
        rowp, colp = P.permanent_ordering(n, cp, ri, rp, ci)
        B = A[np.ix_(rowp, colp)]
        cpb, rib, _, _ = csr_csc(B)
        k, c = P.partitioning(n, cpb, rib)
        # Fig. 3a: bottom-left region empty
        assert not np.any(B[k:, :c])
        ks_ord.append(k)
        ks_raw.append(k_raw)
    assert np.mean(ks_ord) <= np.mean(ks_raw)   # Fig. 4 trend


def test_gray_code_definition():
    """Gray_g = g XOR (g >> 1): a bijection on [0, 2^k) whose
    consecutive codes differ in exactly one bit, the bit ctz(g) (Alg. 1 line 9)."""
    k = 10
    codes = [P.gray(g) for g in range(1 << k)]
    assert sorted(codes) == list(range(1 << k))
    for g in range(1, 1 << k):
        d = codes[g] ^ codes[g - 1]
        assert d & (d - 1) == 0 and d == g & -g


def test_degree_sort_properties():
    """Sec. VI-B degree sort: a permutation whose column degrees are
    nondecreasing, equal degrees in ascending index."""
    A = synth.erdos_renyi(30, 0.2, 4)
    cp, ri, _ = synth.to_ccs(A)
    order = P.degree_sort_ascending(30, cp)
    assert sorted(order) == list(range(30))
    deg = [(A[:, j] != 0).sum() for j in order]
    for a, b, da, db in zip(order, order[1:], deg, deg[1:]):
        assert da < db or (da == db and a < b)
