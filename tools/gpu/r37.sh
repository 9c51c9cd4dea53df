set -x
timeout 900 python -m pytest tests/test_gpu_fetch.py tests/test_gpu_kv.py tests/test_gpu_vllm_adapter.py -q -m gpu > gpurun_out/r37_tests.log 2>&1; tail -3 gpurun_out/r37_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-phi --no-churn --no-host-compare > gpurun_out/r37_bench.json 2> gpurun_out/r37_bench.err; echo rc=$?
