# v56 (single-CTA reservation shortcut on): GPU suite, smoke, C3/C2/C4 bench lines
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 1200 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 600 python bench.py --workload c2x --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2x.json 2>/dev/null; cat gpurun_out/bench_c2x.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 4 -c 1 \
  -o gpurun_out/prof_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c3.log 2>&1
