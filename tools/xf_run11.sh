# K=9 at the default geometry (B=8, found by scoring the elimination search at
# B=9) and K=8 B=10 U=5 (2^16 tasks), with spills and body-read-only values in
# volatile shared memory, vs the bench kernel.
#   gpurun -- 'bash tools/xf_run11.sh'
O=gpurun_out/xf11.jsonl; : > $O
python tools/kernel_xform.py --variants base --reps 5 >> $O 2>gpurun_out/xf11.err
PERM_SCORE_B=9 PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --plan-kw '{"block_log2":4}' --variants base,ro6,ro12,ro35 --reps 5 >> $O 2>>gpurun_out/xf11.err
PERM_SCORE_B=9 PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --variants base,ro12 --reps 5 >> $O 2>>gpurun_out/xf11.err
PERM_TASK_BITS=16 PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --variants base,ro6,ro12 --reps 5 >> $O 2>>gpurun_out/xf11.err
cat $O; tail -3 gpurun_out/xf11.err
