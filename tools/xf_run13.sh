# spill policy knobs: smem_ro threshold (PERM_SMEM_RO) x tolerance (PERM_SPILL_OK)
O=gpurun_out/spill_ab2.jsonl; : > $O
for cfg in "6 64" "12 64" "6 96" "12 128"; do set -- $cfg
  PERM_SMEM_RO=$1 PERM_SPILL_OK=$2 python tools/spill_ab.py ro$1_ok$2 C2,C3,C4,"seed 2","seed 5",C5 >> $O 2>>gpurun_out/spill_ab2.err
done
cat $O; tail -3 gpurun_out/spill_ab2.err
