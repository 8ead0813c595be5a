import sys, json, time
sys.path.insert(0, '/root/repo')
import synth, paper_2501_15126_b200 as pb
A = synth.erdos_renyi(48, 0.2, 1)
t = time.time()
P = pb.Plan.from_dense(A, mode="reg")
pl = time.time() - t
i = P.info
r = P.compute_ex()
print(json.dumps({"tag": sys.argv[1], "K": i["K"], "B": i["B"], "U": i["U"], "w": i["w_plan"], "spill": i["local_bytes"], "plan_s": pl, "sweep_ms": r.sweep_ms, "value": r.value}), flush=True)
