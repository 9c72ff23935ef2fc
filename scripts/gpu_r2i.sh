# profile build: steps per point and per-segment cycles of the expanded workloads
set -x
for w in c2x.0 c2x.1 meshx.0 meshx.1 c2; do
  FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_prof.so timeout 600 python scripts/ab.py child prof $w 4 1 2>&1 | grep -E "FLPROF|ms" | tail -3
done
