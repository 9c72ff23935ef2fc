# compute-sanitizer on the lean variants and their second pass
set -x
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py lean > gpurun_out/san/san_${tool}_lean.log 2>&1; echo "$tool lean rc=$?"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py cluster9 > gpurun_out/san/san_${tool}_cluster9.log 2>&1; echo "$tool cluster9 rc=$?"
done
