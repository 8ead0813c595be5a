# Round-2 GPU stage B: ncu captures (launch lists, DP audits, --set full) of the
# bench kernel, the plain Alg. 1 sweep, the INT01 n=40 and complex band n=44 kernels.
#   gpurun --timeout 3600 -- 'bash tools/gpu_ncu2.sh TAG'
TAG=${1:-r2}
M=sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-cold"
# bench: launch list of whole steps, DP audit + full capture of the sweep
timeout 600 ncu --nvtx --nvtx-include bench_step/ --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cold --no-plain > /dev/null 2>&1; echo launches rc=$?
timeout 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include bench_step/ -k regex:perm_sweep -c 1 --csv --log-file gpurun_out/${TAG}_dpaudit.csv $B --no-plain > /dev/null 2>&1; echo audit rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include bench_step/ -k regex:perm_sweep -c 1 -o gpurun_out/${TAG}_full $B --no-plain > /dev/null 2>&1; echo full rc=$?
# plain Alg. 1 sweep (bench's plain leg)
timeout 900 ncu --metrics $M --clock-control none --nvtx --nvtx-include plain_step/ -k regex:perm_sweep -c 1 --csv --log-file gpurun_out/${TAG}_plain_dpaudit.csv $B > /dev/null 2>&1; echo plain audit rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include plain_step/ -k regex:perm_sweep -c 1 -o gpurun_out/${TAG}_plain_full $B > /dev/null 2>&1; echo plain full rc=$?
# INT01 0/1 n=40 and complex band n=44
for W in int01_n40 complex_band44; do
  timeout 300 python tools/kernel_probe.py $W > gpurun_out/${TAG}_probe_$W.json 2>gpurun_out/${TAG}_probe_$W.err; echo probe $W rc=$?
  timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include probe_step/ -k regex:perm_sweep -c 1 -o gpurun_out/${TAG}_${W}_full python tools/kernel_probe.py $W --reps 1 > /dev/null 2>&1; echo ncu $W rc=$?
done
ls -la gpurun_out/ | grep $TAG
