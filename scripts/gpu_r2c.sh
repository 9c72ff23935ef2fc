set -x
timeout 900 python -m pytest tests/test_topo.py -m gpu -x -q 2>&1 | tail -5
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 900 python scripts/ab.py run --workload c4dp --points 148 --reps 3 v41 base 2>&1 | tail -2
timeout 900 python scripts/ab.py run --workload c4fsdp --points 148 --reps 3 v41 base 2>&1 | tail -2
timeout 900 python scripts/ab.py run --points 1184 --reps 5 v41 base 2>&1 | tail -2
