set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_churn.py -q -m gpu -x > gpurun_out/r84_t.log 2>&1; tail -3 gpurun_out/r84_t.log
timeout 1200 python bench.py --no-cpu-baseline --no-kv > gpurun_out/r84_bench.json 2> gpurun_out/r84_bench.err; echo rc=$?; tail -3 gpurun_out/r84_bench.err
