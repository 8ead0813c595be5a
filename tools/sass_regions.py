"""Map ncu's per-SASS-instruction stall samples (``--page source --csv
--print-source sass``) to the regions of the generated kernel (seed, block
loop, switch case j, block body, tail) using the cubin's line table
(``nvdisasm -gi``, call-site lines for inlined helpers).

    python tools/sass_regions.py SASS.csv KERNEL.cu KERNEL.cubin
"""
from __future__ import annotations

import collections
import csv
import re
import subprocess
import sys


def main():
    csv_path, src_path, cubin = sys.argv[1:4]
    rows = list(csv.reader(open(csv_path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    H = rows[h]
    R = [dict(zip(H, r)) for r in rows[h + 1:] if len(r) == len(H)]
    dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    lines, cur = [], None
    for l in dis.split("\n"):
        m = re.findall(r"line (\d+)", l) if "## File" in l else None
        if m:
            cur = int(m[-1])
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+", l):
            lines.append(cur)
    assert len(lines) == len(R), (len(lines), len(R))
    src = open(src_path).read().split("\n")
    cases = [(i + 1, int(m.group(1))) for i, l in enumerate(src) for m in [re.match(r"\s+case (\d+): \{", l)] if m]
    loop = next(i + 1 for i, l in enumerate(src) if "for (unsigned blk" in l)
    body = max(i + 1 for i, l in enumerate(src) if "default: break;" in l) + 2
    tail = max(i + 1 for i, l in enumerate(src) if re.search(r"\blacc\b", l) and "=" in l)

    def region(line):
        if line is None:
            return "none"
        if line < loop:
            return "seed"
        if line >= tail:
            return "tail"
        if line >= body:
            return "body"
        r = "loop"
        for b, j in cases:
            if line >= b:
                r = f"case{j}"
        return r
    reasons = [x for x in H if x.startswith("stall_") and "Not Issued" not in x]
    agg = collections.defaultdict(collections.Counter)
    for d, ln in zip(R, lines):
        g = region(ln)
        op = d["Source"].split()[0].split(".")[0]
        ex = int(d["Instructions Executed"] or 0)
        agg[g]["exec"] += ex
        agg[g]["op_" + op] += ex
        for r in reasons:
            agg[g][r[6:]] += int(d[r] or 0)
    def samples(c):
        return sum(v for k, v in c.items() if k != "exec" and not k.startswith("op_"))
    tot = sum(samples(c) for c in agg.values())
    for g, c in sorted(agg.items(), key=lambda kv: -samples(kv[1])):
        s = samples(c)
        top = sorted(((v, k) for k, v in c.items() if k != "exec" and not k.startswith("op_")), reverse=True)[:5]
        ops = sorted(((v, k[3:]) for k, v in c.items() if k.startswith("op_")), reverse=True)[:4]
        print(f"{g:8s} samples {s / tot:6.1%} exec {c['exec']:12d}  " + ", ".join(f"{k} {v / s:.0%}" for v, k in top)
              + "  | " + ", ".join(f"{k} {v / max(1, c['exec']):.0%}" for v, k in ops))


if __name__ == "__main__":
    main()
