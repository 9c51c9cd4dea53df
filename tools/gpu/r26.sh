set -x
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r26_tests.log 2>&1; tail -3 gpurun_out/r26_tests.log
python __graft_entry__.py 2>&1 | tail -1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r26_bench.json 2> gpurun_out/r26_bench.err; echo rc=$?; tail -3 gpurun_out/r26_bench.err
