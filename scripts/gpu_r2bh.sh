# narrow variants' own-lane fields in registers: extended set (base: OCC_CP, FIN, CPMAX, COMP..PEAK),
# first set (regf: COMP..PEAK), none (noregf); then the GPU suite and the C2/C3 bench on base
set -x
python scripts/ab.py run --workload c2 --points 256 --reps 15 base regf noregf
python scripts/ab.py run --workload c2x --points 256 --reps 3 base noregf
python scripts/ab.py run --workload c3 --points 1184 --reps 5 base noregf
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2>/dev/null; cat gpurun_out/bench_c2.json
timeout 600 python bench.py > gpurun_out/bench_c3.json 2>/dev/null; cat gpurun_out/bench_c3.json
timeout 600 python bench.py --workload c2x --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2x.json 2>/dev/null; cat gpurun_out/bench_c2x.json
timeout 900 python bench.py --workload meshx --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_meshx.json 2>/dev/null; cat gpurun_out/bench_meshx.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv \
  python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c2 python scripts/ab.py child base c2 256 1 > gpurun_out/prof_c2.log 2>&1
