# round 2, first call: C4 parity, 2-rank bench test, C4 + C3 bench, full GPU suite
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_c4.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_c4.log; cat gpurun_out/pytest_c4.log
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
timeout 900 python -m pytest tests/test_bench_multi.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_multi.log; cat gpurun_out/pytest_multi.log
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
