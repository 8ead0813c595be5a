# spill tolerance for INT01 and complex (strict by default): model pick and autotune
O=gpurun_out/spill_ab3.jsonl; : > $O
for W in complex_band44 int01_n40 int01_n36 int01_band44; do
  for ok in 0 64 128; do
    for at in -1 0; do
      echo "{\"spill_ok\": $ok, \"autotune\": $at, \"probe\": $(PERM_SPILL_OK=$ok timeout 600 python tools/kernel_probe.py $W --autotune $at 2>>gpurun_out/spill_ab3.err)}" >> $O
    done
  done
done
cat $O; tail -3 gpurun_out/spill_ab3.err
