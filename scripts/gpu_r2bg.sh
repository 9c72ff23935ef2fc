# narrow variants (64/256-lane planes): busy and memory fields in registers (regf) vs shared-memory planes (base)
set -x
python scripts/ab.py run --workload c2 --points 256 --reps 15 regf base
python scripts/ab.py run --workload c2x --points 256 --reps 3 regf base
python scripts/ab.py run --workload meshx --points 128 --reps 2 regf base
python scripts/ab.py run --workload c3 --points 296 --reps 3 regf base
FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_regf.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "race or lean or batched or sweep" 2>&1 | tail -2
