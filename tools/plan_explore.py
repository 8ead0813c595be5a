"""Planner-knob exploration on one workload (GPU): each setting runs in its own
process (the knobs are read from the environment at plan time), plans the
matrix, times perm_compute, and prints W_plan, registers and ms.

    python tools/plan_explore.py [--dim 40] [--p 0.2] [--seed 1]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SETTINGS = [
    {},
    {"PERM_ELIM_CANDS": "12"},
    {"PERM_ELIM_BEAM": "3"},
    {"PERM_ELIM_MAXSIZE": "128"},
    {"PERM_ELIM_MAXSIZE": "160", "PERM_ELIM_CANDS": "10"},
    {"PERM_NO_CC": "1"},
    {"PERM_NO_FUSE": "1"},
]

CHILD = r"""
import json, os, sys, time
sys.path.insert(0, %r)
import synth, paper_2501_15126_b200 as pb
A = synth.erdos_renyi(%d, %r, %d)
kw = json.loads(%r)
t0 = time.time()
P = pb.Plan.from_dense(A, mode="reg", device=0, **kw)
plan_s = time.time() - t0
P.compute()
ms = []
for _ in range(3):
    r = P.compute_ex()
    ms.append(P.last_timing()[0])
i = P.info
print(json.dumps({"w_plan": i["w_plan"], "K": i["K"], "B": i["B"], "U": i["U"], "regs": i["regs_per_thread"],
                  "sweep_ms": min(ms), "plan_s": plan_s, "value": r.value}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=40)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--extra", default="", help="JSON list of extra {env..., '_kw': {...}} settings")
    a = ap.parse_args()
    settings = SETTINGS + (json.loads(a.extra) if a.extra else [])
    for st in settings:
        env = {k: v for k, v in st.items() if not k.startswith("_")}
        kw = st.get("_kw", {})
        code = CHILD % (ROOT, a.dim, a.p, a.seed, json.dumps(kw))
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                             env={**os.environ, **env}, timeout=900)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr.strip()[-300:]
        print(json.dumps({"setting": st}), line, flush=True)


if __name__ == "__main__":
    main()
