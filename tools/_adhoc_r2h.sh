bash tools/gpu_suite.sh r2h build smoke tests
python tools/check_overlap_probe.py > gpurun_out/r2h_check_overlap.json 2>&1; echo probe rc=$?
timeout 1500 python bench.py --steps 10 --warmup 3 --no-kv --no-churn --no-sweep > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo bench rc=$?
