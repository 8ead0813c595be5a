"""Strong-scaling estimate on one GPU: time the whole permanent and each of
the R shards a world of R GPUs would run (same plan, same kernel), report
the implied R-GPU time max_r t_r and efficiency t_1 / (R * max_r t_r)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
import paper_2501_15126_b200 as pb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", dest="n", type=int, default=40)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--worlds", default="2,4,8")
    a = ap.parse_args()
    A = synth.erdos_renyi(a.n, a.p, a.seed)
    P = pb.Plan.from_dense(A, autotune=-1)  # the bench's model pick
    P.compute()
    t1 = min(P.compute_ex().sweep_ms for _ in range(3))
    full = P.compute()
    for R in [int(x) for x in a.worlds.split(",")]:
        ts, parts = [], []
        for r in range(R):
            best = None
            for _ in range(2):
                s = P.shard(r, R)
                best = s if best is None or s.sweep_ms < best.sweep_ms else best
            ts.append(best.sweep_ms)
            parts.append(best)
        f = P.fold(parts)
        print(json.dumps({"R": R, "t1_ms": t1, "max_shard_ms": max(ts), "min_shard_ms": min(ts),
                          "eff": t1 / (R * max(ts)), "bitwise_equal": f.value == full,
                          "tasks": P.info["tasks"]}), flush=True)


if __name__ == "__main__":
    main()
