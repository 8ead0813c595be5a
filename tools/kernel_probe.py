"""Run one named workload's permanent a few times inside an NVTX range, for
ncu captures of kernels the bench does not time (INT01, complex, the plain
Alg. 1 sweep) and for their own CUDA-event timings.

    python tools/kernel_probe.py int01_n40 [--reps 3]
    ncu --nvtx --nvtx-include probe_step/ -k regex:perm_sweep -c 1 --set full ... \
        python tools/kernel_probe.py int01_n40

Prints one JSON line: plan geometry, sweep ms (plan events, min over reps),
result, and (for INT01) the exact value.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOADS = {
    "int01_n40": (lambda: synth.erdos_renyi(40, 0.2, 1, binary=True), dict(mode="int01")),
    "complex_band44": (lambda: synth.unitary_brickwork(44, 4, 1), dict()),
    "plain_n40": (lambda: synth.erdos_renyi(40, 0.2, 1), dict(mode="reg", factor_cols=-1)),
    "plain_n36_hybrid": (lambda: synth.erdos_renyi(36, 0.2, 1), dict(mode="hybrid", factor_cols=-1)),
    "plain_n40_hybrid": (lambda: synth.erdos_renyi(40, 0.2, 1), dict(mode="hybrid", factor_cols=-1)),
    "plain_n36": (lambda: synth.erdos_renyi(36, 0.2, 1), dict(mode="reg", factor_cols=-1)),
    "bench_n40": (lambda: synth.erdos_renyi(40, 0.2, 1), dict(mode="reg")),
    "c2_n30": (lambda: synth.erdos_renyi(30, 0.3, 1), dict(mode="reg")),
    "c3_n36": (lambda: synth.erdos_renyi(36, 0.2, 1), dict(mode="reg")),
    "c3_n36_hybrid": (lambda: synth.erdos_renyi(36, 0.2, 1), dict(mode="hybrid")),
    "c5_band44_hybrid": (lambda: synth.givens_brickwork(44, 4, 1), dict(mode="hybrid")),
    "int01_band44": (lambda: (synth.givens_brickwork(44, 4, 1) != 0).astype(float), dict(mode="int01")),
    "int01_n36": (lambda: synth.erdos_renyi(36, 0.2, 1, binary=True), dict(mode="int01")),
    "band44": (lambda: synth.givens_brickwork(44, 4, 1), dict(mode="reg")),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name", choices=sorted(WORKLOADS))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ordering", default="auto")
    ap.add_argument("--autotune", type=int, default=-1)
    ap.add_argument("--dump", default="", help="directory: write the plan's kernel source and cubin there")
    a = ap.parse_args()
    import torch
    import paper_2501_15126_b200 as pb
    make, kw = WORKLOADS[a.name]
    A = make()
    P = pb.Plan.from_dense(A, a.ordering, device=0, autotune=a.autotune, **kw)
    i = P.info
    if a.dump:
        os.makedirs(a.dump, exist_ok=True)
        open(os.path.join(a.dump, a.name + ".cu"), "w").write(P.source)
        open(os.path.join(a.dump, a.name + ".cubin"), "wb").write(P.cubin())
    P.compute_ex()  # warm-up
    best, r = None, None
    for _ in range(a.reps):
        torch.cuda.nvtx.range_push("probe_step")
        r = P.compute_ex()
        torch.cuda.nvtx.range_pop()
        best = r.sweep_ms if best is None else min(best, r.sweep_ms)
    out = {"workload": a.name, "n": i["n"], "mode": i["mode"], "K": i["K"], "B": i["B"], "U": i["U"], "M": i["M"],
           "tasks": i["tasks"], "nnz": i["nnz"], "w_plan": i["w_plan"], "w_alg1": i["w_alg1"],
           "regs": i["regs_per_thread"], "blocks_per_sm": i["blocks_per_sm"], "swept_order": i["swept_order"],
           "tier_rows": i["tier_rows"], "sweep_ms": best, "value": r.value, "value_im": r.value_im,
           "gray_steps": r.steps}
    if r.exact_valid:
        out["exact"] = str(r.exact())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
