set -x
timeout 600 python -m pytest tests/test_gpu_vllm_adapter.py -q -m gpu > gpurun_out/r12_tests.log 2>&1; tail -25 gpurun_out/r12_tests.log
