# A/B: narrow-plane variants with their own register budget (base) vs 64 registers (wide)
set -x
python scripts/ab.py run --workload c2 --points 256 --reps 5 wide base
python scripts/ab.py run --workload c2x.0 --points 128 --reps 3 wide base
python scripts/ab.py run --workload c2x.1 --points 128 --reps 3 wide base
python scripts/ab.py run --workload meshx.0 --points 128 --reps 3 wide base
