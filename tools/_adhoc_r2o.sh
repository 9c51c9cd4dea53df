bash tools/gpu_suite.sh r2o build file:tests/test_gpu_decode.py
timeout 1500 python bench.py --steps 5 --warmup 3 --no-kv --no-churn --no-sweep --no-cpu-baseline > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err; echo bench rc=$?; tail -2 gpurun_out/r2o_bench.err | cut -c1-300
