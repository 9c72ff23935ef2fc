# collective arrivals: a two-REDUX uniform check before __match_any_sync (matchx) vs match only (base)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 matchx base
python scripts/ab.py run --workload c2 --points 256 --reps 15 matchx base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 matchx base
python scripts/ab.py run --workload c4dp --points 270 --reps 3 matchx base
