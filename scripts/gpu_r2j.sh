# message phase with per-thread message registers, in-flight entries carry their reservation
set -x
timeout 1200 python -m pytest tests/test_expanded_scale.py tests/test_expand.py -m gpu -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "p2p or corpus or cluster" 2>&1 | tail -2
for w in c2x.0 meshx.0 meshx.1; do
  FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_prof.so timeout 600 python scripts/ab.py child prof $w 4 1 2>&1 | grep -E "FLPROF|ms" | tail -2
done
timeout 900 python bench.py --workload c2x --steps 10 --warmup 3 > gpurun_out/bench_c2x.json 2> gpurun_out/bench_c2x.err; cat gpurun_out/bench_c2x.json; tail -3 gpurun_out/bench_c2x.err
timeout 900 python bench.py --workload meshx --steps 5 --warmup 3 > gpurun_out/bench_meshx.json 2> gpurun_out/bench_meshx.err; cat gpurun_out/bench_meshx.json; tail -3 gpurun_out/bench_meshx.err
