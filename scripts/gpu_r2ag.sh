# lean single-CTA variants with every lane a rank (no `active` tests) vs with them
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 nofull base
python scripts/ab.py run --workload c2 --points 256 --reps 9 nofull base
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -k "batched or north_star or race or sweep" 2>&1 | tail -3
