# ncu --set full captures of the cluster variant (C4 dp and fsdp families) and of C2
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c4dp python scripts/ab.py child base c4dp 148 1 > gpurun_out/prof_c4dp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c4fsdp python scripts/ab.py child base c4fsdp 148 1 > gpurun_out/prof_c4fsdp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c2 python scripts/ab.py child base c2 256 1 > gpurun_out/prof_c2.log 2>&1
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
tail -3 gpurun_out/*.log
