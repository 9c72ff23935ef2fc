# lean: warp-uniform collective arrivals skip __match_any_sync (vs always matching)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 nouni base
python scripts/ab.py run --workload c2 --points 256 --reps 9 nouni base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 nouni base
