"""Calibration sweep (GPU): sweep-kernel time vs (factored columns K, chunk
bits B, threads per block) on the bench workloads.  Prints one JSON line per
configuration: W_plan, registers, blocks/SM, sweep ms, achieved FP64 lane-op
rate and Gray steps/s.  Used to fit the planner's occupancy/work trade-off."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
import paper_2501_15126_b200 as pb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=36)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--seeds", default="1,2")
    ap.add_argument("--ks", default="-1,2,4,6")
    ap.add_argument("--bs", default="8,10,12")
    ap.add_argument("--threads", default="128")
    ap.add_argument("--minb", default="0")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    for seed in [int(s) for s in a.seeds.split(",")]:
        A = synth.erdos_renyi(a.n, a.p, seed) if a.p > 0 else synth.givens_brickwork(a.n, 4, seed)
        for k in [int(s) for s in a.ks.split(",")]:
            for b in [int(s) for s in a.bs.split(",")]:
              for th in [int(s) for s in a.threads.split(",")]:
                for mb in [int(s) for s in a.minb.split(",")]:
                    try:
                        P = pb.Plan.from_dense(A, mode="reg", factor_cols=k, chunk_log2=b, threads_per_block=th,
                                               min_blocks=mb)
                    except pb.PermError as e:
                        print(json.dumps({"seed": seed, "K": k, "B": b, "err": str(e)[:120]}), flush=True)
                        continue
                    i = P.info
                    P.compute()
                    ms = []
                    for _ in range(a.reps):
                        r = P.compute_ex()
                        ms.append(r.sweep_ms)
                    sw = min(ms)
                    steps = 2 ** (a.n - 1)
                    rate = i["w_plan"] * steps / (sw / 1e3)
                    print(json.dumps({"n": a.n, "seed": seed, "Kreq": k, "minb": mb, "K": i["K"], "B": i["B"],
                                      "U": i["U"], "order": i["ordering"], "var": i["swept_order"],
                                      "M": i["M"], "threads": th, "regs": i["regs_per_thread"],
                                      "bps": i["blocks_per_sm"], "warps_per_smsp": i["blocks_per_sm"] * th / 128,
                                      "w_plan": round(i["w_plan"], 4), "live": i["reg_rows"],
                                      "sweep_ms": round(sw, 3), "steps_per_s": steps / (sw / 1e3),
                                      "tops": rate / 1e12, "frac": rate / (148 * 64 * 1.965e9),
                                      "value": r.value}), flush=True)
                    P.close()


if __name__ == "__main__":
    main()
