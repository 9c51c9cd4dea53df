set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_fetch.py -q -m gpu -x > gpurun_out/r7_tests.log 2>&1; tail -30 gpurun_out/r7_tests.log
