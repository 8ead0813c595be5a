import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2501_15126_b200 as pb
A = synth.erdos_renyi(40, 0.2, 1)
for kw in [dict(no_device=True), dict(device=0), dict(device=0, block_log2=5, min_blocks=1)]:
    P = pb.Plan.from_dense(A, mode='reg', **kw)
    i = P.info
    print(kw, {k: i[k] for k in ('K', 'B', 'U', 'w_plan', 'regs_per_thread', 'local_bytes')}, flush=True)
    P.close()
print([l.strip() for l in open('/proc/self/maps') if 'nvrtc' in l or 'ptx' in l.lower()][:6])
