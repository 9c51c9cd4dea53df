set -x
timeout 900 python -m pytest tests/test_gpu_fetch.py tests/test_gpu_decode.py -q -m gpu -x > gpurun_out/r46_tests.log 2>&1; tail -4 gpurun_out/r46_tests.log
timeout 600 python tools/il_probe.py > gpurun_out/r46_il.json 2> gpurun_out/r46_il.err; tail -3 gpurun_out/r46_il.err
