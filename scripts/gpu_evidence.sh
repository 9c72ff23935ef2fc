# full evidence pass for one engine version: GPU tests, smoke, every bench line, the reference
# arm, launch list and ncu --set full captures of C3, C2 and the C4 families.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 1200 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 600 python bench.py --workload c2x --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2x.json 2> gpurun_out/bench_c2x.err; cat gpurun_out/bench_c2x.json
timeout 900 python bench.py --workload meshx --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_meshx.json 2> gpurun_out/bench_meshx.err; cat gpurun_out/bench_meshx.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv \
  python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 4 -c 1 \
  -o gpurun_out/prof_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c2 python scripts/ab.py child base c2 256 1 > gpurun_out/prof_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c4dp python scripts/ab.py child base c4dp 148 1 > gpurun_out/prof_c4dp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c4fsdp python scripts/ab.py child base c4fsdp 148 1 > gpurun_out/prof_c4fsdp.log 2>&1
ls -la gpurun_out
