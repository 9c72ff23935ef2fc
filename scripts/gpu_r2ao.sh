# clusters without messages: fenced arrivals + L1-bypassing reads instead of a cluster barrier per completion step
set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_c4.py -x -q -k "cluster or c4 or C4" 2>&1 | tail -3
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 clsync base
python scripts/ab.py run --workload c4dp --points 270 --reps 3 clsync base
