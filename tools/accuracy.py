"""FP64 accuracy probe (GPU): relative error of several kernel variants
against the long-double oracle on ER matrices, with kappa = sum|terms|/|perm|."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402  (test infrastructure: accuracy measurement only)
import synth  # noqa: E402
import paper_2501_15126_b200 as pb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="24,28,32")
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--seeds", default="1,2")
    a = ap.parse_args()
    variants = {"K0_B12": dict(factor_cols=-1, chunk_log2=12), "K0_B8": dict(factor_cols=-1, chunk_log2=8),
                "auto": dict(), "hyb_K0": dict(mode="hybrid", factor_cols=-1)}
    for n in [int(x) for x in a.ns.split(",")]:
        for seed in [int(x) for x in a.seeds.split(",")]:
            A = synth.erdos_renyi(n, a.p, seed)
            exp, sabs = oracle.perm_nw(A)
            row = {"n": n, "seed": seed, "kappa": sabs / abs(exp)}
            for name, kw in variants.items():
                kw = dict(kw)
                kw.setdefault("mode", "reg")
                P = pb.Plan.from_dense(A, **kw)
                v = P.compute()
                row[name] = abs(v - exp) / abs(exp)
                row[name + "_K"] = P.info["K"]
                P.close()
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
