# single-CTA points skip the second step reduction after a full-world reservation (rs1) vs not (base)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 rs1 base
python scripts/ab.py run --workload c2 --points 256 --reps 15 rs1 base
python scripts/ab.py run --workload c2x --points 256 --reps 3 rs1 base
FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_rs1.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_c4.py tests/test_expanded_scale.py tests/test_passes.py -x -q 2>&1 | tail -1
