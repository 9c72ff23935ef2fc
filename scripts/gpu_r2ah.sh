# probe: lean variants that assume folding and no host-stream nodes (upper bound of that specialization)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 base probe
python scripts/ab.py run --workload c2 --points 256 --reps 9 base probe
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 base probe
