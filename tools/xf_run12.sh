# planner policy A/B: strict spill gate (round-2 default) vs spill tolerance + smem_ro rung
#   gpurun -- 'bash tools/xf_run12.sh'
O=gpurun_out/spill_ab.jsonl; : > $O
PERM_SPILL_OK=0 PERM_NO_SMEM_RO=1 python tools/spill_ab.py strict >> $O 2>gpurun_out/spill_ab.err
python tools/spill_ab.py tolerant >> $O 2>>gpurun_out/spill_ab.err
PERM_SCORE_B=9 python tools/spill_ab.py tolerant_b9 >> $O 2>>gpurun_out/spill_ab.err
cat $O; tail -3 gpurun_out/spill_ab.err
