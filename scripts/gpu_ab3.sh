timeout 900 python scripts/ab.py run --points 1184 --reps 5 base "$@" 2>&1 | tail -8
FLINT_B200_LIB=$PWD/paper_2604_17550_b200/_build/ab_$1.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o gpurun_out/prof_ab_$1 python scripts/ab.py child $1 c3 1184 1 > gpurun_out/prof_ab.log 2>&1
tail -2 gpurun_out/prof_ab.log
