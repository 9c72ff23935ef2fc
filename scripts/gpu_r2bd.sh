# compute-sanitizer on the 8-stream variant and on the lean pass with the deferred second pass
set -x
python scripts/sanitize.py streams8
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py streams8 > gpurun_out/san_${tool}_streams8.log 2>&1; tail -3 gpurun_out/san_${tool}_streams8.log
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py lean > gpurun_out/san_memcheck_lean.log 2>&1; tail -3 gpurun_out/san_memcheck_lean.log
