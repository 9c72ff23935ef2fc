# L1 warm-up of small graphs' node records and edge lists (base) vs none (nopf)
set -x
python scripts/ab.py run --workload c2 --points 256 --reps 15 base nopf
python scripts/ab.py run --workload c2x --points 256 --reps 3 base nopf
python scripts/ab.py run --workload c3 --points 1184 --reps 5 base nopf
python scripts/ab.py run --workload c4fsdp --points 270 --reps 3 base nopf
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -k "batched or north_star or lean or cluster_8192 or sweep or fsdp2048" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 4 -c 1 \
  -o gpurun_out/prof_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c3.log 2>&1
