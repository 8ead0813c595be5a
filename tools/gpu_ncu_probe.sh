# ncu --set full + per-SASS source page of one probe workload, with its kernel dump
#   gpurun -- 'bash tools/gpu_ncu_probe.sh TAG WORKLOAD'
TAG=$1; W=$2
python tools/kernel_probe.py $W ${PROBE_ARGS} --dump gpurun_out/dump_$TAG > gpurun_out/${TAG}_probe.json 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include probe_step/ -k regex:perm_sweep -c 1 -o gpurun_out/${TAG}_full python tools/kernel_probe.py $W ${PROBE_ARGS} --reps 1 > /dev/null 2>&1; echo ncu rc=$?
ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
cat gpurun_out/${TAG}_probe.json
