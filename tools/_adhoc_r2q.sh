bash tools/gpu_suite.sh r2q build
python tools/d2h_probe.py > gpurun_out/r2q_d2h.json 2>&1; echo d2h rc=$?
timeout 1500 python bench.py --steps 3 --warmup 3 --no-churn --no-sweep --no-cpu-baseline > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err; echo bench rc=$?
