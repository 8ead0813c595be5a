python tools/kernel_xform.py --variants base,br1 --reps 7 > gpurun_out/xf4.jsonl 2>gpurun_out/xf4.err
python tools/kernel_xform.py --dim 36 --variants base,br1 --reps 7 >> gpurun_out/xf4.jsonl 2>>gpurun_out/xf4.err
python tools/kernel_xform.py --variants base,br1 --plan-kw '{"factor_cols": -1, "ordering": "permanent"}' --reps 3 >> gpurun_out/xf4.jsonl 2>>gpurun_out/xf4.err
cat gpurun_out/xf4.jsonl | cut -c1-200; tail -3 gpurun_out/xf4.err
