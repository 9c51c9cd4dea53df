set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py -q -m gpu -x > gpurun_out/r53_tests.log 2>&1; tail -30 gpurun_out/r53_tests.log
timeout 600 python tools/fused_probe.py > gpurun_out/r53_fused.json 2> gpurun_out/r53_fused.err; echo rc=$?; tail -5 gpurun_out/r53_fused.err
