"""Small permanents through every kernel flavour, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck) runs on a B200:

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py

FP64 plain sweep and column-eliminated sweep, the HYBRID global tier, INT01
(block / warp-task zero skip), complex, a 2-shard fold, spilling FP64 (with
volatile shared-memory body reads) and INT01 kernels, a shard of the bench
plan, and a structurally singular input (no launch).  Each result is checked against the oracle."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: the checker)
import synth  # noqa: E402
import paper_2501_15126_b200 as pb  # noqa: E402


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def main():
    A = synth.erdos_renyi(18, 0.3, 1)
    exp, _ = oracle.perm_nw(A)
    for kw in (dict(mode="reg", factor_cols=-1), dict(mode="reg"), dict(mode="hybrid", factor_cols=-1)):
        P = pb.Plan.from_dense(A, **kw)
        v = P.compute()
        assert rel(v, exp) < 1e-9, (kw, v, exp)
        print("ok", kw, P.info["K"], P.info["tier_rows"], flush=True)
        if kw == dict(mode="reg"):
            s = [P.shard(r, 2) for r in range(2)]
            f = P.fold(s)
            assert f.value == v, (f.value, v)
            print("ok shards", flush=True)
        P.close()
    B = synth.erdos_renyi(16, 0.25, 2, binary=True)
    Q = pb.Plan.from_dense(B, mode="int01")
    assert Q.exact() == oracle.perm_nw_exact(B)
    print("ok int01", flush=True)
    Z = synth.unitary_brickwork(16, 3, 1)
    R = pb.Plan.from_dense(Z)
    r = R.compute_ex()
    ez = oracle.perm_band_complex(Z, synth.half_bandwidth(Z))
    assert abs(complex(r.value, r.value_im) - ez) <= 1e-9 * abs(ez)
    print("ok complex", flush=True)
    # DESIGN 3.13(f): a spilling FP64 kernel that reads body values from
    # volatile shared-memory slots (the smem_ro rung, forced), and a spilling
    # INT01 kernel (accepted under autotune in production)
    os.environ.update(PERM_SMEM_RO_FORCE="1", PERM_SPILL_OK="4096", PERM_ELIM_TIER4="0")
    C = synth.erdos_renyi(22, 0.3, 2)
    P = pb.Plan.from_dense(C, mode="reg", block_log2=5, autotune=-1)
    assert P.info["local_bytes"] > 0 and "volatile double" in P.source
    assert rel(P.compute(), oracle.perm_nw(C)[0]) < 1e-9
    print("ok fp64 spill + smem_ro", P.info["local_bytes"], flush=True)
    del os.environ["PERM_SMEM_RO_FORCE"]
    os.environ["PERM_SPILL_OK"] = "64"
    D = synth.erdos_renyi(26, 0.25, 3, binary=True)
    Q = pb.Plan.from_dense(D, mode="int01", block_log2=4, autotune=-1)
    assert Q.info["local_bytes"] > 0
    assert Q.exact() == oracle.perm_nw_exact(D)
    print("ok int01 spill", Q.info["local_bytes"], flush=True)
    del os.environ["PERM_SPILL_OK"]
    del os.environ["PERM_ELIM_TIER4"]
    # the bench plan (n=40, K=8 B=8 U=5, 48-byte frame): one 1/128 shard
    E = synth.erdos_renyi(40, 0.2, 1)
    P = pb.Plan.from_dense(E, mode="reg", autotune=-1)
    r = P.shard(0, 128)
    assert r.value == r.value  # not NaN: the partial is checked against the oracle in tests/
    print("ok bench plan shard", P.info["K"], P.info["U"], P.info["local_bytes"], flush=True)
    S = A.copy()
    S[:, 3] = 0
    S[:, 5] = 0
    S[2, 3] = 0.5
    T = pb.Plan.from_dense(S)
    assert T.compute() == 0.0
    print("ok singular", flush=True)


if __name__ == "__main__":
    main()
