set -x
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_fetch.py -q -m gpu -k "kv_gather_parity or irregular or many_descriptors" > gpurun_out/r15_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r15_memcheck.log; tail -5 gpurun_out/r15_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_target.py kv tma 1 > gpurun_out/r15_racecheck_tma.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r15_racecheck_tma.log; tail -3 gpurun_out/r15_racecheck_tma.log
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/profile_target.py hbm tma 1 > gpurun_out/r15_synccheck_tma.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/r15_synccheck_tma.log; tail -3 gpurun_out/r15_synccheck_tma.log
for spec in "kv tma" "hbm tma" "kv ldg256"; do set -- $spec; timeout 300 ncu --set full --clock-control none --import-source on -k regex:"copy" -c 2 -o gpurun_out/r15_prof_$1_$2 -f python tools/profile_target.py $1 $2 2 > /dev/null 2>&1; done
ls gpurun_out | grep r15
