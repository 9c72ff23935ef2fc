# usage: bash scripts/gpu_ab.sh CANDIDATE [other variants...]: parity tests on the candidate build, then A/B timing
cand=$1; shift
FLINT_B200_LIB=$PWD/paper_2604_17550_b200/_build/ab_$cand.so timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/ab_pytest_$cand.log
cat gpurun_out/ab_pytest_$cand.log
timeout 900 python scripts/ab.py run --points 1184 --reps 5 base $cand "$@" 2>&1 | tail -12
