TAG=$1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo bench rc=$?
timeout 600 ncu --nvtx --nvtx-include bench_step/ --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu1.log 2>&1; echo ncu rc=$?
timeout 600 ncu --metrics sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum --clock-control none --nvtx --nvtx-include bench_step/ -k regex:perm_sweep -c 1 --csv --log-file gpurun_out/${TAG}_dpaudit.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1; echo audit rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include bench_step/ -k regex:perm_sweep -c 1 -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu3.log 2>&1; echo ncufull rc=$?
tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
