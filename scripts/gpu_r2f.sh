# round 2: parallel message phase -- expanded parity, expanded bench lines + ncu, sanitizer logs
set -x
timeout 1200 python -m pytest tests/test_expanded_scale.py tests/test_expand.py -m gpu -x -q 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "p2p or corpus or race" 2>&1 | tail -3
timeout 900 python bench.py --workload c2x --steps 10 --warmup 3 > gpurun_out/bench_c2x.json 2> gpurun_out/bench_c2x.err; cat gpurun_out/bench_c2x.json; tail -3 gpurun_out/bench_c2x.err
timeout 900 python bench.py --workload meshx --steps 10 --warmup 3 > gpurun_out/bench_meshx.json 2> gpurun_out/bench_meshx.err; cat gpurun_out/bench_meshx.json; tail -3 gpurun_out/bench_meshx.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2x.csv \
  python bench.py --workload c2x --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_c2x.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 6 -c 2 \
  -o gpurun_out/prof_c2x python bench.py --workload c2x --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c2x.log 2>&1
for tool in memcheck racecheck synccheck; do
  for case in analytical p2p; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py $case > gpurun_out/san_${tool}_${case}.log 2>&1; echo "$tool $case rc=$?"
  done
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize.py cluster > gpurun_out/san_memcheck_cluster.log 2>&1; echo "memcheck cluster rc=$?"
ls -la gpurun_out
