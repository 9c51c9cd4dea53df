set -x
timeout 900 python -m pytest tests/test_gpu_fetch.py -q -m gpu > gpurun_out/r35_tests.log 2>&1; tail -2 gpurun_out/r35_tests.log
timeout 600 python tools/fetch_microbench.py > gpurun_out/r35_micro.json 2> gpurun_out/r35_micro.err; tail -2 gpurun_out/r35_micro.err
