# clock64 section profile (-DFL_PROFILE, warp 0 of CTA 0): event steps per point and cycles per section
set -x
FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_prof.so python scripts/ab.py child prof c2 256 1 2>&1 | grep -a FLPROF | tail -1
FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_prof.so python scripts/ab.py child prof c3 148 1 2>&1 | grep -a FLPROF | tail -1
