python tools/kernel_xform.py --variants base,pipej,br1 --reps 7 > gpurun_out/xf6.jsonl 2>gpurun_out/xf6.err
python tools/kernel_xform.py --workload complex_band44 --variants base,pipej,br1 --reps 5 >> gpurun_out/xf6.jsonl 2>>gpurun_out/xf6.err
python tools/kernel_xform.py --workload c3_n36 --variants base,pipej --reps 7 >> gpurun_out/xf6.jsonl 2>>gpurun_out/xf6.err
python tools/kernel_xform.py --workload band44 --variants base,pipej --reps 7 >> gpurun_out/xf6.jsonl 2>>gpurun_out/xf6.err
python tools/kernel_xform.py --variants base,pipej --plan-kw '{"factor_cols": -1, "ordering": "permanent"}' --reps 3 >> gpurun_out/xf6.jsonl 2>>gpurun_out/xf6.err
cut -c1-200 gpurun_out/xf6.jsonl; tail -3 gpurun_out/xf6.err
