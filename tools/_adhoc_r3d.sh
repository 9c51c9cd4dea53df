bash tools/gpu_suite.sh r3d build
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_fetch_hook.py -q -m gpu -k "not k2_phi35 and not k1_config1" > gpurun_out/r3d_memcheck_fetch.log 2>&1; echo "memcheck fetch rc=$?"; tail -3 gpurun_out/r3d_memcheck_fetch.log
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -k "trailing or tokens_shorter or fused_in_place" > gpurun_out/r3d_memcheck_attn.log 2>&1; echo "memcheck attn rc=$?"; tail -3 gpurun_out/r3d_memcheck_attn.log
timeout 1500 $CS --tool racecheck --error-exitcode 9 python tools/profile_target.py attn ldg 1 > gpurun_out/r3d_racecheck_attn.log 2>&1; echo "racecheck attn rc=$?"; tail -2 gpurun_out/r3d_racecheck_attn.log
timeout 1500 $CS --tool synccheck --error-exitcode 9 python tools/profile_target.py attn ldg 1 > gpurun_out/r3d_synccheck_attn.log 2>&1; echo "synccheck attn rc=$?"; tail -2 gpurun_out/r3d_synccheck_attn.log
timeout 1500 $CS --tool racecheck --error-exitcode 9 python tools/profile_target.py checked ldg16 1 > gpurun_out/r3d_racecheck_checked.log 2>&1; echo "racecheck checked rc=$?"; tail -2 gpurun_out/r3d_racecheck_checked.log
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_ipc.py -q -m gpu > gpurun_out/r3d_memcheck_ipc.log 2>&1; echo "memcheck ipc rc=$?"; tail -3 gpurun_out/r3d_memcheck_ipc.log
