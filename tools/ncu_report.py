"""Summarise round-2 ncu captures into profiles/.

    python tools/ncu_report.py --round r2 --tag g3

Reads gpurun_out/<tag>_launches.csv (bench launch list), <tag>_dpaudit.csv /
<tag>_full.ncu-rep (bench sweep), <tag>_plain_dpaudit.csv / <tag>_plain_full.ncu-rep
(plain Alg. 1 sweep), <tag>_<w>_full.ncu-rep + <tag>_probe_<w>.json for the
probe workloads (INT01 n=40, complex band n=44).  Writes
profiles/<round>_kernel_ncu.json (per-plan audit entries bench.py matches by
plan signature: executed DP instructions per Gray step, DRAM bytes per
launch) and prints markdown tables for profiles/<round>_ncu_summary.md.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from ncu_summary import KEYS, full_metrics, launch_shares, num  # noqa: E402

EXTRA = [
    ("smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst executed"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe cycles active"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe"),
    ("smsp__sass_thread_inst_executed_op_integer_pred_on.sum", "integer thread-instructions"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-instructions"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread-instructions"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
]

WORKLOADS = {
    "bench": (lambda s: s.erdos_renyi(40, 0.2, 1), dict(mode="reg", autotune=-1), "auto"),
    "plain": (lambda s: s.erdos_renyi(40, 0.2, 1), dict(mode="reg", autotune=-1, factor_cols=-1), "permanent"),
    "int01_n40": (lambda s: s.erdos_renyi(40, 0.2, 1, binary=True), dict(mode="int01", autotune=-1), "auto"),
    "complex_band44": (lambda s: s.unitary_brickwork(44, 4, 1), dict(autotune=-1), "auto"),
}


def signature(name):
    import synth
    import paper_2501_15126_b200 as pb
    make, kw, order = WORKLOADS[name]
    P = pb.Plan.from_dense(make(synth), order, no_device=True, **kw)
    i = P.info
    import hashlib
    i = dict(i, kernel_sha=hashlib.sha256(P.source.encode()).hexdigest()[:16])
    P.close()
    return {k: i[k] for k in ("n", "nnz", "K", "B", "U", "M", "tasks", "w_plan")}, i


def dp_count(path):
    dp = 0.0
    for r in csv.reader(open(path)):
        if len(r) > 3 and "perm_sweep" in " ".join(r) and "_pred_on.sum" in " ".join(r):
            dp += float(r[-1].replace(",", ""))
    return dp


def table(k):
    rows = []
    for m, label in KEYS + EXTRA:
        if m in k:
            rows.append(f"| {label} (`{m}`) | {k[m][1]} {k[m][0]} |")
    return "\n".join(["| metric | value |", "|---|---|"] + rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r2")
    ap.add_argument("--tag", default="g3")
    a = ap.parse_args()
    g = os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    out_entries = []
    md = []
    lp = os.path.join(g, f"{a.tag}_launches.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(prof, f"{a.round}_launches_bench.csv"))
        md.append("### Launch list (bench steps)\n\n| kernel | launches | total ms | share | avg ms |\n|---|---:|---:|---:|---:|")
        for k, cnt, ms, share, avg in launch_shares(lp):
            md.append(f"| {k} | {cnt} | {ms:.3f} | {100 * share:.2f} % | {avg:.4f} |")
    for name, rep, audit in (("bench", f"{a.tag}_full.ncu-rep", f"{a.tag}_dpaudit.csv"),
                             ("plain", f"{a.tag}_plain_full.ncu-rep", f"{a.tag}_plain_dpaudit.csv"),
                             ("int01_n40", f"{a.tag}_int01_n40_full.ncu-rep", None),
                             ("complex_band44", f"{a.tag}_complex_band44_full.ncu-rep", None)):
        rp = os.path.join(g, rep)
        if not os.path.exists(rp):
            continue
        ks = [k for k in full_metrics(rp) if "perm_sweep" in k.get("Kernel Name", ("", ""))[1]]
        if not ks:
            continue
        k = ks[0]
        sig, info = signature(name)
        gray = info["tasks"] * 32 * info["M"] * (1 << info["B"]) * (1 << info["K"])
        e = {"workload": name, "signature": sig, "kernel_sha": info["kernel_sha"],
             "dram_bytes_per_launch": num(k["dram__bytes_read.sum"]) + num(k["dram__bytes_write.sum"]),
             "source": f"profiles/{a.round}_ncu_summary.md (ncu --set full, {rep})",
             "fp64_pipe_pct": num(k["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
             "kernel_ms": num(k["gpu__time_duration.sum"]) / 1e6 if k["gpu__time_duration.sum"][0] in ("ns", "nsecond")
             else num(k["gpu__time_duration.sum"]),
             "registers": num(k["launch__registers_per_thread"])}
        dpp = os.path.join(g, audit) if audit else None
        if dpp and os.path.exists(dpp):
            dp = dp_count(dpp)
            shutil.copy(dpp, os.path.join(prof, f"{a.round}_dpaudit_{name}.csv"))
        else:  # the --set full capture carries the same thread-instruction counters
            dp = sum(num(k[m]) or 0 for m in ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
                                               "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
                                               "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum") if m in k)
        if dp:
            e["dp_thread_inst_per_launch"] = dp
            e["w_exec"] = dp / gray
            e["w_exec_over_w_plan"] = e["w_exec"] / info["w_plan"]
        out_entries.append(e)
        md.append(f"\n### `{name}`: n={info['n']} mode={info['mode']} K={info['K']} B={info['B']} U={info['U']} "
                  f"W_plan={info['w_plan']:.5f} ({rep})\n")
        md.append(table(k))
        md.append("\n```json\n" + json.dumps(e) + "\n```")
    json.dump({"entries": out_entries}, open(os.path.join(prof, f"{a.round}_kernel_ncu.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
