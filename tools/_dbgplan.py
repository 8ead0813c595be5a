import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2501_15126_b200 as pb
A=synth.erdos_renyi(40,0.2,1)
for kw in [dict(), dict(block_log2=5, min_blocks=1)]:
    for nd in [True, False]:
        P=pb.Plan.from_dense(A, mode='reg', no_device=nd, **kw)
        i=P.info; print(kw, nd, {k:i[k] for k in ('K','B','U','w_plan','regs_per_thread','local_bytes')}, flush=True)
        P.close()
