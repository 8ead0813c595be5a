"""A/B of planner policies on the real-FP64 configs (one GPU): run once per
policy (environment knobs are read per process), model pick (no autotune),
sweep ms = min of 3 plan-event timings after one warm-up.

    PERM_SPILL_OK=0 PERM_NO_SMEM_RO=1 python tools/spill_ab.py strict
    python tools/spill_ab.py default
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
import paper_2501_15126_b200 as pb  # noqa: E402

WORK = [("C2 n=30 p=0.3", lambda: synth.erdos_renyi(30, 0.3, 1)),
        ("C3 n=36 p=0.2", lambda: synth.erdos_renyi(36, 0.2, 1)),
        ("n=36 p=0.2 seed 2", lambda: synth.erdos_renyi(36, 0.2, 2)),
        ("C4 n=40 p=0.2", lambda: synth.erdos_renyi(40, 0.2, 1)),
        ("n=40 p=0.2 seed 2", lambda: synth.erdos_renyi(40, 0.2, 2)),
        ("n=40 p=0.2 seed 3", lambda: synth.erdos_renyi(40, 0.2, 3)),
        ("n=40 p=0.2 seed 4", lambda: synth.erdos_renyi(40, 0.2, 4)),
        ("n=40 p=0.2 seed 5", lambda: synth.erdos_renyi(40, 0.2, 5)),
        ("C5 n=44 band depth 4", lambda: synth.givens_brickwork(44, 4, 1)),
        ("n=44 band U(0,1]", lambda: synth.band_positive(44, 4, 1))]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "run"
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    for name, make in WORK:
        if only and not any(o in name for o in only):
            continue
        A = make()
        if A is None:
            continue
        P = pb.Plan.from_dense(A, mode="reg", autotune=-1)
        P.compute_ex()
        ms = min(P.compute_ex().sweep_ms for _ in range(3))
        i = P.info
        print(json.dumps({"policy": tag, "config": name, "K": i["K"], "B": i["B"], "U": i["U"], "w_plan": i["w_plan"],
                          "regs": i["regs_per_thread"], "local_bytes": i["local_bytes"], "smem_bytes": i["smem_bytes"],
                          "ms": ms, "value": P.compute(), "plan_ms": i["plan_ms"]}), flush=True)
        P.close()


if __name__ == "__main__":
    main()
