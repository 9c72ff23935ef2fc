# Engine.run fast path for rows-only calls: GPU suite + C2 e2e
set -x
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_e2e_$i.json 2>/dev/null; cat gpurun_out/bench_c2_e2e_$i.json; done
python scripts/e2e_probe.py c2 400
