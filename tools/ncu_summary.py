"""Summarise the bench's ncu captures into profiles/.

    python tools/ncu_summary.py --round r1 --launches gpurun_out/launches.csv \
        --full gpurun_out/bench_full.ncu-rep [--dim 40 --p 0.2 --seed 1 --mode reg]

Writes profiles/<round>_launches_bench.csv (the raw launch list),
profiles/<round>_bench_kernel_ncu.json (per-launch DRAM traffic of the sweep
kernel + its plan signature, read by bench.py for roofline.traffic) and prints
a markdown table of the launch shares and the key `--set full` counters.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEYS = [
    ("gpu__time_duration.sum", "kernel time"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_registers", "blocks / SM (register limit)"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle / issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "stall branch_resolving / issue"),
    ("sass__inst_executed_local_loads", "local loads (spill)"),
    ("sass__inst_executed_local_stores", "local stores (spill)"),
    ("smsp__sass_branch_targets_threads_divergent.sum", "divergent branch targets"),
    ("smsp__sass_branch_targets_threads_uniform.pct", "uniform branch targets"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    unit = "nsecond"
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                unit = d["Metric Unit"]
                name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")[:48]
                agg[name][0] += 1
                agg[name][1] += float(d["Metric Value"].replace(",", ""))
    to_ms = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}[unit]
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append((k, cnt, t * to_ms, t / tot, t * to_ms / cnt))
    return out


def full_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, u = r[0], r[1]
    kernels = []
    for v in r[2:]:
        kernels.append({h[i]: (u[i], v[i]) for i in range(len(h))})
    return kernels


def num(uv):
    u, v = uv
    try:
        return float(v.replace(",", "")) * SCALE.get(u, 1)
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r1")
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--dpaudit", help="ncu csv of the dadd/dmul/dfma thread-instruction counters of one sweep")
    ap.add_argument("--dim", type=int, default=40)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--mode", default="reg")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    if a.launches:
        shutil.copy(a.launches, os.path.join(prof, f"{a.round}_launches_bench.csv"))
        print("| kernel | launches | total ms | share | avg ms |\n|---|---:|---:|---:|---:|")
        for k, cnt, ms, share, avg in launch_shares(a.launches):
            print(f"| {k} | {cnt} | {ms:.3f} | {100 * share:.2f} % | {avg:.4f} |")
    if a.full:
        ks = [k for k in full_metrics(a.full) if "perm_sweep" in k.get("Kernel Name", ("", ""))[1]]
        k = ks[0]
        print("\n| metric | value |\n|---|---|")
        for m, label in KEYS:
            if m in k:
                print(f"| {label} (`{m}`) | {k[m][1]} {k[m][0]} |")
        traffic = num(k["dram__bytes_read.sum"]) + num(k["dram__bytes_write.sum"])
        import synth
        import paper_2501_15126_b200 as pb
        A = synth.erdos_renyi(a.dim, a.p, a.seed)
        P = pb.Plan.from_dense(A, mode=a.mode, no_device=True)
        info = P.info
        sig = {key: info[key] for key in ("n", "nnz", "K", "B", "U", "M", "tasks", "w_plan")}
        P.close()
        out = {"signature": sig, "dram_bytes_per_launch": traffic,
               "source": f"profiles/{a.round}_ncu_summary.md (ncu --set full, {os.path.basename(a.full)})",
               "fp64_pipe_pct": num(k["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
               "kernel_ms": num(k["gpu__time_duration.sum"])}
        if a.dpaudit:
            dp = 0.0
            for r in csv.reader(open(a.dpaudit)):
                if len(r) > 3 and "perm_sweep" in " ".join(r) and "_pred_on.sum" in " ".join(r):
                    dp += float(r[-1].replace(",", ""))
            gray = info["tasks"] * 32 * info["M"] * (1 << info["B"]) * (1 << info["K"])
            out["dp_thread_inst_per_launch"] = dp
            out["w_exec"] = dp / gray
            out["w_exec_over_w_plan"] = out["w_exec"] / info["w_plan"]
            shutil.copy(a.dpaudit, os.path.join(prof, f"{a.round}_dpaudit_bench.csv"))
        path = os.path.join(prof, f"{a.round}_bench_kernel_ncu.json")
        entries = json.load(open(path)).get("entries", []) if os.path.exists(path) else []
        entries = [e for e in entries if e.get("signature") != sig] + [out]  # one entry per audited plan
        json.dump({"entries": entries}, open(path, "w"), indent=1)
        print("\n", json.dumps(out))


if __name__ == "__main__":
    main()
