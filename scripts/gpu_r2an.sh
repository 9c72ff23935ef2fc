# lean: `done` bits for tracked consumers only (vs every pop)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 notrack base
python scripts/ab.py run --workload c2 --points 256 --reps 9 notrack base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 notrack base
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
