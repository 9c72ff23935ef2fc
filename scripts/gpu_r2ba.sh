# warp min of step keys by two REDUX (redux) vs the lockstep shortcut + shuffle tree (base)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 redux base
python scripts/ab.py run --workload c2 --points 256 --reps 15 redux base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 redux base
python scripts/ab.py run --workload c2x --points 256 --reps 3 redux base
