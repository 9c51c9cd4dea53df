set -x
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/r11_smoke.log 2>&1; tail -2 gpurun_out/r11_smoke.log
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/r11_tests.log 2>&1; tail -25 gpurun_out/r11_tests.log
