python tools/kernel_xform.py --variants base,asap,alap,rand3 --reps 7 > gpurun_out/xf7.jsonl 2>gpurun_out/xf7.err
python tools/kernel_xform.py --workload c3_n36 --variants base,asap,alap --reps 7 >> gpurun_out/xf7.jsonl 2>>gpurun_out/xf7.err
python tools/kernel_xform.py --workload complex_band44 --variants base,asap,alap --reps 5 >> gpurun_out/xf7.jsonl 2>>gpurun_out/xf7.err
python tools/kernel_xform.py --workload band44 --variants base,asap,alap --reps 7 >> gpurun_out/xf7.jsonl 2>>gpurun_out/xf7.err
python tools/kernel_xform.py --workload c2_n30 --variants base,asap,alap --reps 7 >> gpurun_out/xf7.jsonl 2>>gpurun_out/xf7.err
python tools/kernel_xform.py --variants base,asap,alap --plan-kw '{"factor_cols": -1, "ordering": "permanent"}' --reps 3 >> gpurun_out/xf7.jsonl 2>>gpurun_out/xf7.err
python -c "
import json
for l in open('gpurun_out/xf7.jsonl'):
    d=json.loads(l); print(d['variant'], d['regs'], d['spill'], round(d['ms_min'],4), round(d['speedup_vs_base'],4), d['slots_bitwise_equal'], d['K'], d['U'])
"; tail -3 gpurun_out/xf7.err
