# A/B of the codegen post-pass knobs on every probe workload (model-picked plans)
#   gpurun -- 'bash tools/gpu_ab.sh TAG'
#   ENVS="A=1;A=2 B=3" WL="bench_n40 c3_n36" gpurun -- 'bash tools/gpu_ab.sh TAG'
TAG=${1:-ab}
ENVS=${ENVS:-";PERM_NO_KC=1"}
WL=${WL:-bench_n40 c2_n30 c3_n36 c5_band44_hybrid band44 complex_band44 int01_n40 int01_n36 int01_band44}
IFS=';' read -ra EL <<< "$ENVS"
for W in $WL; do
  for E in "${EL[@]}"; do
    echo -n "{\"env\": \"$E\", \"r\": " >> gpurun_out/${TAG}.jsonl
    env $E timeout 600 python tools/kernel_probe.py $W --reps 3 >> gpurun_out/${TAG}.jsonl 2>>gpurun_out/${TAG}.err || echo '{}' >> gpurun_out/${TAG}.jsonl
    sed -i '$ s/$/}/' gpurun_out/${TAG}.jsonl
  done
done
python - <<PY
import json
for l in open("gpurun_out/${TAG}.jsonl"):
    try: d=json.loads(l)
    except Exception: print("bad", l[:200]); continue
    r=d["r"]
    if r: print(f'{r["workload"]:18s} {d["env"]:34s} ms {r["sweep_ms"]:.4f} K {r["K"]} B {r["B"]} U {r["U"]} regs {r["regs"]} bps {r["blocks_per_sm"]} w {r["w_plan"]:.5g}')
PY
