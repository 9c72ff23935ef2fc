# fl_sweep_run launches the lean variant's second pass only when a status it read back is FL_RETRY
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lean_pass" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 > gpurun_out/bench_c2_$i.json 2>/dev/null; cat gpurun_out/bench_c2_$i.json; done
python scripts/e2e_probe.py c2 400 > gpurun_out/e2e_probe_c2.txt 2>&1; cat gpurun_out/e2e_probe_c2.txt
timeout 600 python bench.py > gpurun_out/bench_c3.json 2>/dev/null; cat gpurun_out/bench_c3.json
