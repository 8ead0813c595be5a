# validation after the planner restructuring (Planner class) and the INT01 spill policy
TAG=g14
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests rc=$?
for W in int01_n40 int01_n36 int01_band44; do timeout 600 python tools/kernel_probe.py $W --autotune 0; done > gpurun_out/${TAG}_int01.jsonl 2>&1
timeout 1200 python tools/time_configs.py > gpurun_out/${TAG}_configs.jsonl 2>gpurun_out/${TAG}_configs.err; echo configs rc=$?
tail -3 gpurun_out/${TAG}_gpu_tests.log; cat gpurun_out/${TAG}_int01.jsonl
