mkdir -p gpurun_out
for v in v0 v1 v2 v3 v4; do HARVEST_B200_LIB=build/ffnvar3/$v.so timeout 300 python tools/fused_probe.py hbm > gpurun_out/r119_$v.json 2> gpurun_out/r119_$v.err; echo $v rc=$?; HARVEST_B200_LIB=build/ffnvar3/$v.so timeout 300 python -m pytest tests/test_gpu_decode.py -q -m gpu -x -k "fused_ffn_kernels" 2>&1 | tail -1; done
