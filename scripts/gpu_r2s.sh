# cl_step_clic: cluster parity (SPMD graphs, forced sizes, C4 goldens), C4 with / without it; C3 ncu
set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_c4.py -x -q 2>&1 | tail -3
FL_NO_CLIC=1 timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_noclic.json 2> gpurun_out/bench_c4_noclic.err; cat gpurun_out/bench_c4_noclic.json
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c3 python scripts/ab.py child base c3 4096 1 > gpurun_out/prof_c3.log 2>&1
tail -2 gpurun_out/prof_c3.log
