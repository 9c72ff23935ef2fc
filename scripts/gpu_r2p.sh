# A/B: offset column views (base) vs HEAD engine (orig), C4 families and C3; cluster parity
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" 2>&1 | tail -2
python scripts/ab.py run --workload c4dp --points 270 --reps 3 orig base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 orig base
python scripts/ab.py run --workload c3 --points 1184 --reps 3 orig base
