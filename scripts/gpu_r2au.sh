# comm FIFO rings sized by the antichain depth bound (vs coll_stride rows) + full GPU suite
set -x
python scripts/ab.py run --workload c3 --points 1184 --reps 5 prev base
python scripts/ab.py run --workload c2 --points 256 --reps 9 prev base
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 prev base
python scripts/ab.py run --workload c4dp --points 270 --reps 3 prev base
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
