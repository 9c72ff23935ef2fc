# lean variant (no event record / trace / shared first-dependency bitmap branches) vs the general one
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 nolean base
python scripts/ab.py run --workload c3 --points 4096 --reps 3 nolean base
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or north_star or batched or sweep" 2>&1 | tail -3
