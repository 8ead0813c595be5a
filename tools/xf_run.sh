python tools/kernel_xform.py --variants base,kc,b64,kc_b64 > gpurun_out/xf1.jsonl 2>gpurun_out/xf1.err
PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --variants base,kc --plan-kw '{"block_log2": 4, "chunk_log2": 9, "factor_cols": 8}' >> gpurun_out/xf1.jsonl 2>>gpurun_out/xf1.err
python tools/kernel_xform.py --variants base,kc --plan-kw '{"factor_cols": -1, "ordering": "permanent"}' >> gpurun_out/xf1.jsonl 2>>gpurun_out/xf1.err
cat gpurun_out/xf1.jsonl; tail -5 gpurun_out/xf1.err
