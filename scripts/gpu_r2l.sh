# zero-copy host path (fl_sweep_run), cached fl_points, permuted-group pairing
set -x
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json
timeout 900 python bench.py --workload c2x --steps 10 --warmup 3 > gpurun_out/bench_c2x.json 2> gpurun_out/bench_c2x.err; cat gpurun_out/bench_c2x.json
timeout 900 python bench.py --workload meshx --steps 5 --warmup 3 > gpurun_out/bench_meshx.json 2> gpurun_out/bench_meshx.err; cat gpurun_out/bench_meshx.json
