set -x
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r100_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r100_bench_ncu.log 2>&1; echo rc=$?; tail -c 300 gpurun_out/r100_bench_ncu.log
