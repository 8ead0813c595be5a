# Round-2 GPU stage C: per-instruction stall sampling of the bench sweep
# (source page), HYBRID tier vs shared-memory placement at K=0 (timings + full
# captures of the tier kernels).
#   gpurun --timeout 3600 -- 'bash tools/gpu_ncu3.sh TAG'
TAG=${1:-g5}
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-cold --no-plain"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include bench_step/ -k regex:perm_sweep -c 1 -o gpurun_out/${TAG}_full $B > /dev/null 2>&1; echo full rc=$?
ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_full_sass.csv 2>gpurun_out/${TAG}_sass.err; echo sass rc=$?
for W in plain_n36 plain_n36_hybrid plain_n40 plain_n40_hybrid; do
  timeout 300 python tools/kernel_probe.py $W > gpurun_out/${TAG}_probe_$W.json 2>gpurun_out/${TAG}_probe_$W.err; echo probe $W rc=$?
done
for W in plain_n36_hybrid plain_n36; do
  timeout 1200 ncu --set full --clock-control none --nvtx --nvtx-include probe_step/ -k regex:perm_sweep -c 1 -o gpurun_out/${TAG}_${W}_full python tools/kernel_probe.py $W --reps 1 > /dev/null 2>&1; echo ncu $W rc=$?
done
cat gpurun_out/${TAG}_probe_*.json
ls -la gpurun_out/ | grep $TAG
