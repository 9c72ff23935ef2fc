# one ncu --set full capture of the C3 sweep kernel + the launch list of the bench command
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
  -o gpurun_out/prof_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
  -o gpurun_out/prof_c4 python bench.py --workload c4 --points 296 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c4.log 2>&1
ls -la gpurun_out
