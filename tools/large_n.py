"""Record-scale runs on one GPU: larger sparse / banded
permanents, timed with the plan's CUDA events, resumable via checkpoint.py."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
import paper_2501_15126_b200 as pb  # noqa: E402
from paper_2501_15126_b200.checkpoint import compute_resumable  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ckdir", default="gpurun_out")
    a = ap.parse_args()
    cases = [("ER n=44 p=0.2", synth.erdos_renyi(44, 0.2, 1)),
             ("ER n=48 p=0.2", synth.erdos_renyi(48, 0.2, 1)),
             ("band n=54 depth 4 (boson sampling)", synth.givens_brickwork(54, 4, 1)),
             ("complex unitary band n=54 depth 4", synth.unitary_brickwork(54, 4, 1))]
    for name, A in cases:
        n = A.shape[0]
        t0 = time.perf_counter()
        P = pb.Plan.from_dense(A)
        plan_s = time.perf_counter() - t0
        i = P.info
        ck = os.path.join(a.ckdir, f"ck_{n}_{i['mode']}.json")
        if os.path.exists(ck):
            os.remove(ck)
        t0 = time.perf_counter()
        r = compute_resumable(P, ck)  # auto_pieces: >= 2^14 warp-tasks per piece
        wall = time.perf_counter() - t0
        sweep = 0.0
        import json as _j
        for d in _j.load(open(ck))["done"].values():
            sweep += d["sweep_ms"]
        print(json.dumps({"case": name, "n": n, "mode": i["mode"], "K": i["K"], "B": i["B"], "w_plan": i["w_plan"],
                          "regs": i["regs_per_thread"], "plan_s": plan_s, "sweep_s": sweep / 1e3, "wall_s": wall,
                          "gray_steps_per_s": (2 ** (n - 1) - 1) / (sweep / 1e3),
                          "value": r.value, "value_im": r.value_im}), flush=True)


if __name__ == "__main__":
    main()
