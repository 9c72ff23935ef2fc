# cluster occupancy probe; ncu --set full of C2 and of both C4 families (cluster variant); C2 bench (NVML clocks)
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_clusters scripts/probe_clusters.cu && /tmp/probe_clusters > gpurun_out/probe_clusters.txt; cat gpurun_out/probe_clusters.txt | head -120
timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c2 python scripts/ab.py child base c2 256 1 > gpurun_out/prof_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c4dp python scripts/ab.py child base c4dp 144 1 > gpurun_out/prof_c4dp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c4fsdp python scripts/ab.py child base c4fsdp 144 1 > gpurun_out/prof_c4fsdp.log 2>&1
tail -3 gpurun_out/prof_*.log
