# message-phase statistics (rounds per phase) on the expanded workloads; fresh C3 ncu + launch list
set -x
for w in meshx.0 meshx.1 c2x.0 c2x.1; do
  FLINT_B200_LIB=paper_2604_17550_b200/_build/ab_msgstat.so timeout 600 python scripts/ab.py child msgstat $w 8 1 2>&1 | grep -E "FLMSG|name" | tail -2
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
  -o gpurun_out/prof_c3 python scripts/ab.py child base c3 4096 1 > gpurun_out/prof_c3.log 2>&1
tail -2 gpurun_out/prof_c3.log
