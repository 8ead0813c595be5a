python tools/kernel_xform.py --variants base,hot2,vol,hot2+vol,hot2+ro,hot2+ro+lb3,ro+lb2 > gpurun_out/xf3.jsonl 2>gpurun_out/xf3.err
python tools/kernel_xform.py --variants base,hot2+ro,hot2+ro+lb3 --plan-kw '{"block_log2": 4, "chunk_log2": 9, "factor_cols": 8}' >> gpurun_out/xf3.jsonl 2>>gpurun_out/xf3.err
python tools/kernel_xform.py --variants base,hot2,hot2+ro,hot2+ro+lb4 --plan-kw '{"factor_cols": -1, "ordering": "permanent"}' >> gpurun_out/xf3.jsonl 2>>gpurun_out/xf3.err
cat gpurun_out/xf3.jsonl; tail -5 gpurun_out/xf3.err
