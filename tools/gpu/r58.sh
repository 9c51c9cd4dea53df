set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r58_smoke.log 2>&1; tail -1 gpurun_out/r58_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r58_tests.log 2>&1; tail -2 gpurun_out/r58_tests.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_decode.py -q -m gpu -x -k fused > gpurun_out/r58_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r58_memcheck.log; tail -3 gpurun_out/r58_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_target.py fused x 1 > gpurun_out/r58_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r58_racecheck.log; tail -3 gpurun_out/r58_racecheck.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"expert_ffn" -c 2 -o gpurun_out/r58_prof_fused -f python tools/profile_target.py fused x 1 > gpurun_out/r58_prof.log 2>&1; echo rc=$?
