# A/B: RL from the constant bank (noldg), + ld.global.nc graph tables (base), vs HEAD (prev)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 prev noldg base
python scripts/ab.py run --workload c2 --points 256 --reps 9 prev noldg base
python scripts/ab.py run --workload c4dp --points 270 --reps 3 prev base
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" 2>&1 | tail -3
