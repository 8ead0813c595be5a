python tools/kernel_xform.py --variants base,hot2,hot2c16,hot3 > gpurun_out/xf2.jsonl 2>gpurun_out/xf2.err
python tools/kernel_xform.py --variants base,hot2,hot3 --plan-kw '{"factor_cols": -1, "ordering": "permanent"}' >> gpurun_out/xf2.jsonl 2>>gpurun_out/xf2.err
cat gpurun_out/xf2.jsonl; tail -5 gpurun_out/xf2.err
