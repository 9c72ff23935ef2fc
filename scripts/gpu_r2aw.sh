# lean: no due-set test in next_time, no t > tcur test per step (vs with them)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 nostep base
python scripts/ab.py run --workload c2 --points 256 --reps 9 nostep base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 nostep base
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -k "batched or north_star or lean or cluster_8192 or sweep or fsdp2048" 2>&1 | tail -2
