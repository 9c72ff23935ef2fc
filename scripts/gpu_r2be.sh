# fl_sweep_run completion: cudaStreamSynchronize (FL_SYNC_SPIN=0) vs a cudaStreamQuery spin (1)
set -x
for i in 1 2; do
  FL_SYNC_SPIN=0 python scripts/e2e_probe.py c2 400 2>&1 | head -2
  FL_SYNC_SPIN=1 python scripts/e2e_probe.py c2 400 2>&1 | head -2
done
for s in 0 1 0 1; do FL_SYNC_SPIN=$s timeout 600 python bench.py --workload c2 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('spin', $s, d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['ms_per_step_median'])"; done
