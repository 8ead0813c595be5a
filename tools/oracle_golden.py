"""Write full-size oracle goldens for the bench workloads (calls only oracle/
and synth/; no product code): tests/golden/oracle_<name>.json with the
long-double Alg. 1 permanent (oracle.perm_nw) and sum |terms|.

    python tools/oracle_golden.py [--names c3_n36,c4_n40]

C4 (n=40, 2^39 Gray steps) takes ~40 min on 16 host cores; C3 (n=36) ~2.5 min;
the exact 0/1 n=40 case (c4b_n40_01) ~2.5 h on 8 cores.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

CASES = {
    "c3_n36": ("Erdos-Renyi n=36 p=0.2 seed=1, values U(0,1] (BASELINE configs[2])", lambda: synth.erdos_renyi(36, 0.2, 1)),
    "c4_n40": ("Erdos-Renyi n=40 p=0.2 seed=1, values U(0,1] (BASELINE configs[3], the bench workload)",
               lambda: synth.erdos_renyi(40, 0.2, 1)),
}
# exact integer goldens (0/1 inputs): oracle.perm_nw_exact = Alg. 1 in doubled
# integers, wrapping int128, certified by T' = 0 mod 2^(n-1)
EXACT_CASES = {
    "c4b_n40_01": ("0/1 Erdos-Renyi n=40 p=0.2 seed=1 (the INT01 zero-skip workload, BASELINE configs[3] pattern)",
                   lambda: synth.erdos_renyi(40, 0.2, 1, binary=True)),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--names", default="c3_n36,c4_n40")
    a = ap.parse_args()
    for name in a.names.split(","):
        if name in EXACT_CASES:
            desc, make = EXACT_CASES[name]
            A = make()
            t0 = time.perf_counter()
            v = oracle.perm_nw_exact(A)
            dt = time.perf_counter() - t0
            out = {"case": desc, "n": int(A.shape[0]), "perm_exact": str(v),
                   "oracle": "oracle.perm_nw_exact (Alg. 1 in doubled exact integers, int128, T' divisible by 2^(n-1))",
                   "seconds": round(dt, 1), "threads": oracle.max_threads(), "script": "tools/oracle_golden.py"}
            path = os.path.join(ROOT, "tests", "golden", f"oracle_{name}.json")
            json.dump(out, open(path, "w"), indent=1)
            print(json.dumps(out), flush=True)
            continue
        desc, make = CASES[name]
        A = make()
        t0 = time.perf_counter()
        v, sabs = oracle.perm_nw(A)
        dt = time.perf_counter() - t0
        out = {"case": desc, "n": int(A.shape[0]), "perm": repr(v), "sum_abs_terms": repr(sabs),
               "kappa": sabs / abs(v), "oracle": "oracle.perm_nw (Alg. 1, long double, pairwise chunk fold)",
               "seconds": round(dt, 1), "threads": oracle.max_threads(),
               "script": "tools/oracle_golden.py"}
        path = os.path.join(ROOT, "tests", "golden", f"oracle_{name}.json")
        json.dump(out, open(path, "w"), indent=1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
