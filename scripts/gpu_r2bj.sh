# parked set-member finishes with streaming (evict-first) stores/loads (cpcs) vs default (base)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 cpcs base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 cpcs base
python scripts/ab.py run --workload c4dp --points 270 --reps 3 cpcs base
python scripts/ab.py run --workload c2 --points 256 --reps 15 cpcs base
