# compute-sanitizer on the round-2 kernel changes: 9-CTA clusters, clusters of 600-rank CTAs with messages,
# single-CTA points without the accumulator clear
set -x
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  for case in analytical cluster9 cluster_p2p; do
    timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py $case > gpurun_out/san/san_${tool}_${case}.log 2>&1; echo "$tool $case rc=$?"
  done
done
tail -n 3 gpurun_out/san/*.log
