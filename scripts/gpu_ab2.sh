# usage: bash scripts/gpu_ab2.sh "pytest args" VARIANTS...: one failing-test probe on the first variant, then A/B timing
probe=$1; shift
cand=$1
FLINT_B200_LIB=$PWD/paper_2604_17550_b200/_build/ab_$cand.so timeout 600 python -m pytest $probe -x -q 2>&1 | grep -v '^$' | tail -25
timeout 900 python scripts/ab.py run --points 1184 --reps 5 base "$@" 2>&1 | tail -12
