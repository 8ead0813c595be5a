"""Where the end-to-end (public API, host buffers) time of one n=40 permanent
goes: perm_plan (cache hit) + device setup, sweep + fold, D2H, perm_free.

    python tools/e2e_breakdown.py [--dim 40] [--reps 5]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=40)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch
    import synth
    import paper_2501_15126_b200 as pb
    from paper_2501_15126_b200.dist import ShardedPermanent
    A = synth.erdos_renyi(a.dim, a.p, 1)
    ptr, idx, val = pb.dense_to_ccs(A)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    rows = []
    for k in range(a.reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P = pb.Plan(a.dim, pb.PERM_CCS, ptr, idx, val, "auto", mode="reg", device=0, stream=stream.cuda_stream)
        t1 = time.perf_counter()
        sp = ShardedPermanent(P, 0, 1, dev)
        t2 = time.perf_counter()
        sp.step()
        t3 = time.perf_counter()
        v = sp.value()
        t4 = time.perf_counter()
        plan_ms = P.info["plan_ms"]
        P.close()
        t5 = time.perf_counter()
        rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, plan_ms))
    print("plan+load | buffers | enqueue | sweep+sync+D2H | free | (plan_ms)   [ms]")
    for r in rows[1:]:
        print(" | ".join(f"{1000 * x:8.3f}" for x in r[:5]), f"| {r[5]:.3f}")


if __name__ == "__main__":
    main()
