bash tools/gpu_suite.sh r2f build file:tests/test_gpu_kv_decode.py
python tools/attn_probe.py > gpurun_out/r2f_attn_fused.json 2>&1; echo a rc=$?
HARVEST_B200_LIB=build/attn_2kernel/libharvest_b200.so python tools/attn_probe.py > gpurun_out/r2f_attn_2k.json 2>&1; echo b rc=$?
