python tools/kernel_xform.py --variants base,kcase,kall --reps 7 > gpurun_out/xf5.jsonl 2>gpurun_out/xf5.err
python tools/kernel_xform.py --dim 36 --variants base,kcase,kall --reps 7 >> gpurun_out/xf5.jsonl 2>>gpurun_out/xf5.err
python tools/kernel_xform.py --dim 30 --p 0.3 --variants base,kcase,kall --reps 7 >> gpurun_out/xf5.jsonl 2>>gpurun_out/xf5.err
python tools/kernel_xform.py --variants base,kcase,kall --plan-kw '{"factor_cols": -1, "ordering": "permanent"}' --reps 3 >> gpurun_out/xf5.jsonl 2>>gpurun_out/xf5.err
cut -c1-220 gpurun_out/xf5.jsonl; tail -3 gpurun_out/xf5.err
