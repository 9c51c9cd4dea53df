bash tools/gpu_suite.sh r2w build file:tests/test_gpu_decode.py
python tools/fused_probe.py hbm > gpurun_out/r2w_fused_dyn.json 2>&1; echo dyn rc=$?
HARVEST_B200_LIB=build/ffn_static/libharvest_b200.so python tools/fused_probe.py hbm > gpurun_out/r2w_fused_static.json 2>&1; echo static rc=$?
