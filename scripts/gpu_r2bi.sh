# narrow variants' own-lane fields in registers: all but F_COMM_END (base), F_COMP..F_PEAK only (regf), none (noregf)
set -x
python scripts/ab.py run --workload c2 --points 256 --reps 15 base regf noregf
python scripts/ab.py run --workload c2x --points 256 --reps 3 base regf noregf
python scripts/ab.py run --workload c3 --points 296 --reps 3 base regf noregf
FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_regf.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "race or lean or batched or sweep" 2>&1 | tail -2
