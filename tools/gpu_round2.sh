# Round-2 GPU round-trip, stage A: smoke, GPU tests, bench.  Outputs in gpurun_out/.
#   gpurun --timeout 3600 -- 'bash tools/gpu_round2.sh TAG'
TAG=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests rc=$?
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo bench rc=$?
tail -5 gpurun_out/${TAG}_gpu_tests.log; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-600
