# giant composite tier on by default (real FP64): validation + A/B + bench
bash tools/gpu_round2.sh g19
python tools/spill_ab.py tier4_default > gpurun_out/g19_ab.jsonl 2>gpurun_out/g19_ab.err
python tools/n48_probe.py tier4_default >> gpurun_out/g19_ab.jsonl 2>>gpurun_out/g19_ab.err
cat gpurun_out/g19_ab.jsonl
