# set-member critical-path words through L2 only (cpcg: st.cg/ld.cg, no L1 allocation) vs default (base)
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 cpcg base
python scripts/ab.py run --workload c2 --points 256 --reps 15 cpcg base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 cpcg base
python scripts/ab.py run --workload c4dp --points 270 --reps 3 cpcg base
