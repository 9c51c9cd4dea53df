set -x
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r87_memcheck_all.log 2>&1; echo "memcheck rc=$?"; grep -E "passed|failed|ERROR SUMMARY" gpurun_out/r87_memcheck_all.log | tail -3
