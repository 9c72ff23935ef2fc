# round 2: MinSet member counts (no scans of empty overflow bitmaps)
set -x
timeout 1200 python -m pytest tests/test_expanded_scale.py tests/test_expand.py -m gpu -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --workload c2x --steps 10 --warmup 3 > gpurun_out/bench_c2x.json 2> gpurun_out/bench_c2x.err; cat gpurun_out/bench_c2x.json; tail -3 gpurun_out/bench_c2x.err
timeout 900 python bench.py --workload meshx --steps 10 --warmup 3 > gpurun_out/bench_meshx.json 2> gpurun_out/bench_meshx.err; cat gpurun_out/bench_meshx.json; tail -3 gpurun_out/bench_meshx.err
timeout 900 python scripts/ab.py run --workload c3 --points 1184 --reps 5 base 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
  -o gpurun_out/prof_c2x_ring python scripts/ab.py child base c2x.0 128 4 > gpurun_out/prof_c2x.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
  -o gpurun_out/prof_meshx_ring python scripts/ab.py child base meshx.0 128 4 > gpurun_out/prof_meshx.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
  -o gpurun_out/prof_meshx_mh python scripts/ab.py child base meshx.1 128 4 > gpurun_out/prof_meshx1.log 2>&1
