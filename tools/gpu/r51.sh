set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kv.py -q -m gpu -x > gpurun_out/r51_tests.log 2>&1; tail -3 gpurun_out/r51_tests.log
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_fetch.py tests/test_gpu_kv.py tests/test_gpu_vllm_adapter.py -q -m gpu -x -k "not independence" > gpurun_out/r51_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r51_memcheck.log; tail -4 gpurun_out/r51_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_target.py hbm tma 1 > gpurun_out/r51_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r51_racecheck.log; tail -3 gpurun_out/r51_racecheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_target.py blocks tma 1 > gpurun_out/r51_racecheck_blocks.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r51_racecheck_blocks.log; tail -3 gpurun_out/r51_racecheck_blocks.log
