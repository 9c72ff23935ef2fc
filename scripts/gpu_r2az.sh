# 8-stream kernel variant (compute_streams 5-8): parity vs the oracle, full GPU suite, C3/C2 bench unchanged
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "many_compute_streams or more_than_eight" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2>/dev/null; cat gpurun_out/bench_c3.json
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2>/dev/null; cat gpurun_out/bench_c2.json
