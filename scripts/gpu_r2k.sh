# full GPU suite + expanded-mode evidence (ncu of each family, launch lists) + sanitizers on the message path
set -x
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2x.csv \
  python bench.py --workload c2x --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_c2x.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_meshx.csv \
  python bench.py --workload meshx --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_meshx.log 2>&1
for w in c2x.0 c2x.1 meshx.0 meshx.1; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
    -o gpurun_out/prof_$w python scripts/ab.py child base $w 128 4 > gpurun_out/prof_$w.log 2>&1
done
for tool in memcheck racecheck synccheck; do
  for case in analytical p2p; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py $case > gpurun_out/san_${tool}_${case}.log 2>&1; echo "$tool $case rc=$?"
  done
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize.py cluster > gpurun_out/san_memcheck_cluster.log 2>&1; echo "memcheck cluster rc=$?"
