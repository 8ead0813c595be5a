"""Plan + time a few bench-like workloads on cuda:0 (PERM_DEBUG_PLAN=1 shows the
planner candidates and autotune measurements)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2501_15126_b200 as pb
for name, A, mode in [("fp64 n40", synth.erdos_renyi(40, 0.2, 1), "reg"),
                      ("int01 n40", synth.erdos_renyi(40, 0.2, 1, binary=True), "int01"), ("int01 n40 s2", synth.erdos_renyi(40, 0.2, 2, binary=True), "int01"),
                      ("fp64 n36", synth.erdos_renyi(36, 0.2, 1), "reg")]:
    t = time.time()
    P = pb.Plan.from_dense(A, mode=mode, device=0)
    i = P.info
    P.compute()
    ms = min(P.compute_ex().sweep_ms for _ in range(3))
    print(name, {k: i[k] for k in ("K", "B", "U", "w_plan", "regs_per_thread", "swept_order")}, "plan_s", round(time.time() - t, 1), "ms", ms, flush=True)
