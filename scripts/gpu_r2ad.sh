# lean variants everywhere they apply (C3, C4 clusters, narrow C2, expanded) vs none; full GPU suite
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 nolean base
python scripts/ab.py run --workload c2 --points 256 --reps 9 nolean base
python scripts/ab.py run --workload c4dp --points 270 --reps 3 nolean base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 nolean base
python scripts/ab.py run --workload c2x.0 --points 128 --reps 3 nolean base
python scripts/ab.py run --workload meshx.1 --points 128 --reps 3 nolean base
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
