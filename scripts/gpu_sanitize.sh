# compute-sanitizer over one small launch per kernel family (scripts/sanitize_case.py).
# usage: bash scripts/gpu_sanitize.sh TAG   -> gpurun_out/sanitizer_TAG.log
TAG=${1:-r2}
OUT=gpurun_out/sanitizer_$TAG.log
: > $OUT
timeout 300 python scripts/sanitize_case.py all >> $OUT 2>&1
echo "plain rc=$?" >> $OUT
for tool in memcheck synccheck racecheck initcheck; do
  t0=$(date +%s)
  echo "== $tool" >> $OUT
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python scripts/sanitize_case.py all > gpurun_out/san_$tool.log 2>&1
  rc=$?
  grep -E "ok \(|ERROR SUMMARY|RACECHECK SUMMARY|all ok|Error|error" gpurun_out/san_$tool.log | head -80 >> $OUT
  echo "$tool rc=$rc secs=$(( $(date +%s) - t0 ))" >> $OUT
done
