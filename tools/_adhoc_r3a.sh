bash tools/gpu_suite.sh r3a build file:tests/test_gpu_decode.py
python tools/fused_probe.py hbm > gpurun_out/r3a_fused_pair.json 2>&1; echo pair rc=$?
HARVEST_B200_LIB=build/ffn_nopair/libharvest_b200.so python tools/fused_probe.py hbm > gpurun_out/r3a_fused_nopair.json 2>&1; echo nopair rc=$?
