# A/B of the in-tree build against ab_v40, full GPU suite on the in-tree build, C3 bench + ncu
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 900 python scripts/ab.py run --points 1184 --reps 5 v40 base 2>&1 | tail -3
timeout 900 python scripts/ab.py run --workload c4dp --points 148 --reps 3 v40 base 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
  -o gpurun_out/prof_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c3.log 2>&1
ls gpurun_out
