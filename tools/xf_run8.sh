for w in int01_n40 int01_n36 int01_band44; do python tools/kernel_xform.py --workload $w --variants base,m128,m128u --reps 7 >> gpurun_out/xf8.jsonl 2>>gpurun_out/xf8.err; done
python -c "
import json
for l in open('gpurun_out/xf8.jsonl'):
    d=json.loads(l); print(d['variant'], d['regs'], d['spill'], round(d['ms_min'],4), round(d['speedup_vs_base'],4), d['slots_bitwise_equal'], d['K'], d['U'])
"; tail -3 gpurun_out/xf8.err
