"""Sweep-kernel time per permanent for the BASELINE configs and binary
variants (one GPU): mode, K, W_plan, registers, ms, Gray steps/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
import paper_2501_15126_b200 as pb  # noqa: E402


def run(name, A, **kw):
    n = A.shape[0]
    P = pb.Plan.from_dense(A, **kw)
    r = P.compute_ex()
    ms = min(P.compute_ex().sweep_ms for _ in range(3))
    i = P.info
    print(json.dumps({"config": name, "n": n, "mode": i["mode"], "K": i["K"], "B": i["B"], "w_plan": i["w_plan"],
                      "U": i["U"], "regs": i["regs_per_thread"],
                      "blocks_per_sm": i["blocks_per_sm"], "tier_rows": i["tier_rows"], "smem_bytes": i["smem_bytes"], "ms": ms, "steps_per_s": (2 ** (n - 1) - 1) / (ms / 1e3),
                      "value": r.value, "exact": r.exact(), "plan_ms": i["plan_ms"]}), flush=True)
    P.close()


def main():
    run("C1 n=10 p=0.3 0/1 int01", synth.erdos_renyi(10, 0.3, 1, binary=True), mode="int01")
    run("C2 n=30 p=0.3", synth.erdos_renyi(30, 0.3, 1), mode="reg")
    # mode=hybrid asks for Alg. 4's register/global split; after column
    # elimination the planner leaves no rows for the tier (tier_rows = 0, see
    # DESIGN 3.5), so the K=0 rows below show the tier itself at work
    run("C3 n=36 p=0.2 mode=hybrid", synth.erdos_renyi(36, 0.2, 1), mode="hybrid")
    run("C3 n=36 p=0.2 mode=hybrid K=0 (global tier populated)", synth.erdos_renyi(36, 0.2, 1), mode="hybrid",
        factor_cols=-1)
    run("C3 n=36 p=0.2 mode=reg K=0 (shared-memory slots)", synth.erdos_renyi(36, 0.2, 1), mode="reg",
        factor_cols=-1)
    run("C3 n=36 p=0.2 reg", synth.erdos_renyi(36, 0.2, 1), mode="reg")
    run("C4 n=40 p=0.2", synth.erdos_renyi(40, 0.2, 1), mode="reg")
    run("C5 n=44 band depth 4", synth.givens_brickwork(44, 4, 1), mode="reg")
    run("C5 n=44 band depth 4 mode=hybrid", synth.givens_brickwork(44, 4, 1), mode="hybrid")
    run("C5' n=44 band U(0,1]", synth.band_positive(44, 4, 1), mode="reg")
    run("0/1 ER n=36 p=0.2 int01", synth.erdos_renyi(36, 0.2, 1, binary=True), mode="int01")
    run("0/1 ER n=36 p=0.2 int01 no zero-skip", synth.erdos_renyi(36, 0.2, 1, binary=True), mode="int01",
        zero_skip=-1)
    run("0/1 ER n=40 p=0.2 int01", synth.erdos_renyi(40, 0.2, 1, binary=True), mode="int01")
    run("0/1 ER n=40 p=0.2 int01 no zero-skip", synth.erdos_renyi(40, 0.2, 1, binary=True), mode="int01",
        zero_skip=-1)
    run("0/1 ER n=40 p=0.1 int01", synth.erdos_renyi(40, 0.1, 2, binary=True), mode="int01")
    run("0/1 ER n=40 p=0.1 int01 no zero-skip", synth.erdos_renyi(40, 0.1, 2, binary=True), mode="int01",
        zero_skip=-1)
    run("0/1 band n=44 w=4 int01", (synth.givens_brickwork(44, 4, 1) != 0).astype(float), mode="int01")
    run("complex unitary brickwork n=44 depth 4", synth.unitary_brickwork(44, 4, 1))
    run("complex ER n=32 p=0.2", synth.erdos_renyi_complex(32, 0.2, 1))
    run("0/1 ER n=36 p=0.2 fp64", synth.erdos_renyi(36, 0.2, 1, binary=True), mode="reg")
    run("n=44 p=0.2", synth.erdos_renyi(44, 0.2, 1), mode="reg")


if __name__ == "__main__":
    main()
