# skip the accumulator-table clear when the first-dependency bitmap is in shared memory; e2e probe
set -x
python scripts/ab.py run --workload c2 --points 256 --reps 15 prev base
python scripts/ab.py run --workload c2x.0 --points 128 --reps 3 prev base
python scripts/ab.py run --workload meshx.1 --points 128 --reps 3 prev base
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "race or p2p or trace or golden" 2>&1 | tail -3
python scripts/e2e_probe.py c2 300
