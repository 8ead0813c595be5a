set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:perm_sweep -c 1 -o gpurun_out/bench_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; echo ncufull rc=$?
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/bench.log | tail -2
