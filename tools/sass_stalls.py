"""Aggregate ncu's per-SASS-instruction source page (``ncu -i X.ncu-rep --page
source --csv --print-source sass``) by opcode: executed warp-instructions and
warp-stall samples by reason, plus the top stalled instructions.

    python tools/sass_stalls.py gpurun_out/g5_full_sass.csv [--top 30]
"""
from __future__ import annotations

import argparse
import collections
import csv


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    H = rows[hdr]
    out = []
    for r in rows[hdr + 1:]:
        if len(r) < len(H):
            continue
        d = dict(zip(H, r))
        src = d["Source"].strip()
        toks = src.split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
        d["op"] = op.split(".")[0]
        out.append(d)
    return H, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    H, rows = load(a.csv)
    reasons = [h for h in H if h.startswith("stall_") and "Not Issued" not in h]
    by_op = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    for d in rows:
        ex = int(d["Instructions Executed"] or 0)
        by_op[d["op"]]["exec"] += ex
        by_op[d["op"]]["samples"] += int(d["# Samples"] or 0)
        for r in reasons:
            v = int(d[r] or 0)
            by_op[d["op"]][r] += v
            tot[r] += v
    allex = sum(c["exec"] for c in by_op.values())
    alls = sum(tot.values())
    print(f"executed warp-instructions {allex}, stall samples {alls}")
    print("samples by reason:", ", ".join(f"{r[6:]} {v / alls:.1%}" for r, v in tot.most_common() if v))
    print(f"{'op':10s} {'exec':>12s} {'exec%':>6s} {'samp%':>6s}  top reasons")
    for op, c in sorted(by_op.items(), key=lambda kv: -kv[1]["exec"])[:a.top]:
        rs = sorted(((c[r], r[6:]) for r in reasons if c[r]), reverse=True)[:4]
        print(f"{op:10s} {c['exec']:12d} {c['exec'] / allex:6.1%} {c['samples'] / alls:6.1%}  "
              + ", ".join(f"{n} {v / max(1, c['samples']):.0%}" for v, n in rs))


if __name__ == "__main__":
    main()
