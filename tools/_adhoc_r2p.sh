bash tools/gpu_suite.sh r2p build file:tests/test_gpu_kv.py,tests/test_gpu_kv_decode.py,tests/test_gpu_vllm_adapter.py,tests/test_gpu_churn.py
timeout 1500 python bench.py --steps 5 --warmup 3 --no-churn --no-sweep --no-cpu-baseline > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo bench rc=$?; tail -2 gpurun_out/r2p_bench.err | cut -c1-300
