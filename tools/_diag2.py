import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import json, os, sys
sys.path.insert(0, %r)
import synth, paper_2501_15126_b200 as pb
A = synth.erdos_renyi(40, 0.2, 1)
P = pb.Plan.from_dense(A, mode="reg", device=0)
i = P.info
print(json.dumps({"w_plan": i["w_plan"], "U": i["U"], "regs": i["regs_per_thread"], "local": i["local_bytes"]}))
''' % ROOT
for k in range(2):
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env={**os.environ, "PERM_DEBUG_PLAN": "1"})
    print("subprocess", k, out.stdout.strip())
    print("\n".join(l for l in out.stderr.splitlines() if "attempt" in l or "built" in l))
exec(code)
