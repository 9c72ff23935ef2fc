# probe: what compile-time fold + no serial mode would add to the lean variants
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 base leanfold
python scripts/ab.py run --workload c2 --points 256 --reps 9 base leanfold
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 base leanfold
