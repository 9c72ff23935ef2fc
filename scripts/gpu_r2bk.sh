# narrow variants read every point parameter in one round trip (hoist) vs two (nohoist): device and e2e
set -x
python scripts/ab.py run --workload c2 --points 256 --reps 15 hoist nohoist
for i in 1 2; do for v in hoist nohoist; do
  FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_$v.so timeout 600 python bench.py --workload c2 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'median', round(d['e2e']['ms_per_step_median'],4))"
done; done
FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_hoist.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "race or lean or batched or sweep" 2>&1 | tail -1
