"""The paper's Table II synthetic grid on one B200: Erdos-Renyi
n in {40, 45, 48} x p in {0.1 .. 0.5}, values U(0,1] (reading R18), seed 1,
one permanent each, timed with the plan's CUDA events.  Prints one JSON line
per cell with the paper's A100 CodeGen-Hybrid time beside ours (context: the
paper's numbers are another machine's).

    python tools/paper_table.py [--max-s 120]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
import paper_2501_15126_b200 as pb  # noqa: E402

# CodeGen-Hybrid, A100 80 GB, FP64, seconds
PAPER = {40: [3.18, 3.94, 4.77, 5.96, 6.51],
         45: [92.06, 93.69, 155.28, 196.25, 251.07],
         48: [741.59, 1059.77, 1361.69, 1906.64, 2023.94]}
PS = [0.1, 0.2, 0.3, 0.4, 0.5]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-s", type=float, default=120.0, help="skip a cell whose 1/64 probe predicts more")
    ap.add_argument("--ns", default="40,45,48")
    a = ap.parse_args()
    for n in [int(x) for x in a.ns.split(",")]:
        for k, p in enumerate(PS):
            A = synth.erdos_renyi(n, p, 1)
            t0 = time.perf_counter()
            P = pb.Plan.from_dense(A, mode="reg")
            plan_s = time.perf_counter() - t0
            i = P.info
            # probe 1/64 of the range (work per task is uniform for FP64)
            parts = 64 if i["tasks"] >= 64 else 1
            P.shard(0, parts)
            probe_ms = P.last_timing()[0]
            est_s = probe_ms * parts / 1000.0
            row = {"n": n, "p": p, "K": i["K"], "B": i["B"], "U": i["U"], "w_plan": i["w_plan"],
                   "regs": i["regs_per_thread"], "plan_s": round(plan_s, 2),
                   "paper_a100_hybrid_s": PAPER[n][k]}
            if est_s > a.max_s:
                row.update({"skipped": f"estimated {est_s:.1f} s > --max-s"})
            else:
                r = P.compute_ex()
                row.update({"ours_s": r.sweep_ms / 1000.0, "value": r.value,
                            "gray_steps_per_s": (2 ** (n - 1) - 1) / (r.sweep_ms / 1000.0),
                            "speedup_vs_paper": PAPER[n][k] / (r.sweep_ms / 1000.0)})
            print(json.dumps(row), flush=True)
            P.close()


if __name__ == "__main__":
    main()
