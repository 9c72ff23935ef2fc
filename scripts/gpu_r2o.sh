# flexible cluster size: parity at forced sizes, C4 at 8 vs automatic (9) CTAs per cluster
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_c4.py -x -q 2>&1 | tail -3
FL_CLUSTER_CTAS=8 timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_cs8.json 2> gpurun_out/bench_c4_cs8.err; cat gpurun_out/bench_c4_cs8.json
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
