# the previous point's device kept in shared memory (4 registers fewer) vs HEAD
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 prev base
python scripts/ab.py run --workload c2 --points 256 --reps 9 prev base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 prev base
