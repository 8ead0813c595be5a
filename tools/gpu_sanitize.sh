# compute-sanitizer over every kernel flavour (tools/sanitize.py); summaries in gpurun_out/
#   gpurun -- 'bash tools/gpu_sanitize.sh TAG'
TAG=${1:-san}
python tools/sanitize.py > gpurun_out/${TAG}_plain.log 2>&1; echo plain rc=$?
for T in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --error-exitcode 9 python tools/sanitize.py > gpurun_out/${TAG}_$T.log 2>&1
  echo $T rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/${TAG}_$T.log | tail -3
done
