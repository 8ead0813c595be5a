# K=9 U=4 (W 0.2231) with loop-carried values moved to volatile shared memory
# until ptxas fits it without spills, vs the bench kernel (K=8 U=4, W 0.2442).
#   gpurun -- 'bash tools/xf_run10.sh'
O=gpurun_out/xf10.jsonl; : > $O
python tools/kernel_xform.py --variants base --reps 5 >> $O 2>gpurun_out/xf10.err
PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --plan-kw '{"block_log2":4,"chunk_log2":9,"factor_cols":10}' --variants base,ro12,rw40_2,rw40_3,rw12_2,rw1000_2 --reps 5 >> $O 2>>gpurun_out/xf10.err
PERM_ALLOW_SPILL=1 python tools/kernel_xform.py --plan-kw '{"block_log2":5,"chunk_log2":9,"factor_cols":8}' --variants base,rw1000_2,rw40_2 --reps 5 >> $O 2>>gpurun_out/xf10.err
cat $O; tail -3 gpurun_out/xf10.err
