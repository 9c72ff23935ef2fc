# warp-serial message phase (base) vs claim rounds (rounds) on the expanded workloads; message parity
set -x
python scripts/ab.py run --workload c2x.0 --points 128 --reps 3 rounds base
python scripts/ab.py run --workload c2x.1 --points 128 --reps 3 rounds base
python scripts/ab.py run --workload meshx.0 --points 128 --reps 2 rounds base
python scripts/ab.py run --workload meshx.1 --points 128 --reps 3 rounds base
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_expanded_scale.py tests/test_expand.py -x -q -k "p2p or expand or golden or matches_reference" 2>&1 | tail -3
