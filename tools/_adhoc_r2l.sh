bash tools/gpu_suite.sh r2l build file:tests/test_gpu_decode.py
python tools/fused_probe.py hbm > gpurun_out/r2l_fused_t2s3.json 2>&1; echo s3 rc=$?
for S in 2 4; do HARVEST_B200_LIB=build/ffn_t2s$S/libharvest_b200.so python tools/fused_probe.py hbm > gpurun_out/r2l_fused_t2s$S.json 2>&1; echo s$S rc=$?; done
