# Spilling U=5 / K=9 plans vs the bench kernel (kernel_xform variants; volatile
# shared-memory slots for body-read-only values to cut the spill).
#   gpurun -- 'bash tools/xf_run9.sh'
O=gpurun_out/xf9.jsonl; : > $O
python tools/kernel_xform.py --variants base --reps 5 >> $O 2>gpurun_out/xf9.err
PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --plan-kw '{"block_log2":5,"chunk_log2":9,"factor_cols":8}' --variants base,vol,ro12,ro35,vol+alap --reps 5 >> $O 2>>gpurun_out/xf9.err
PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --plan-kw '{"block_log2":5,"chunk_log2":9}' --variants base,vol,ro12 --reps 5 >> $O 2>>gpurun_out/xf9.err
PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --plan-kw '{"block_log2":4,"chunk_log2":9,"factor_cols":9}' --variants base,vol,ro12 --reps 5 >> $O 2>>gpurun_out/xf9.err
cat $O; tail -3 gpurun_out/xf9.err
