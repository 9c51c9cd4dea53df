set -x
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r28_tests.log 2>&1; tail -2 gpurun_out/r28_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r28_bench.json 2> gpurun_out/r28_bench.err; echo rc=$?; tail -3 gpurun_out/r28_bench.err
