bash tools/gpu_suite.sh r2k build file:tests/test_gpu_decode.py
python tools/fused_probe.py hbm > gpurun_out/r2k_fused_tma2d.json 2>&1; echo tma2d rc=$?
HARVEST_B200_LIB=build/ffn_cpasync/libharvest_b200.so python tools/fused_probe.py hbm > gpurun_out/r2k_fused_cpasync.json 2>&1; echo cpasync rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expert_ffn -c 2 -o gpurun_out/r2k_ffn -f python tools/profile_target.py fused ldg 1 > gpurun_out/r2k_ncu.log 2>&1; echo ncu rc=$?
