set -x
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/r16_tests.log 2>&1; tail -3 gpurun_out/r16_tests.log
timeout 300 python tools/host_overhead.py > gpurun_out/r16_overhead.json 2> gpurun_out/r16_overhead.err; tail -3 gpurun_out/r16_overhead.err; cat gpurun_out/r16_overhead.json
