set -x
mkdir -p gpurun_out
for w in 2 4 8; do HARVEST_B200_LIB=build/attnvar2/lib_w$w.so timeout 300 python tools/attn_probe.py > gpurun_out/r102_w$w.json 2> gpurun_out/r102_w$w.err; echo w$w rc=$?; HARVEST_B200_LIB=build/attnvar2/lib_w$w.so timeout 300 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x -k kernel_matches 2>&1 | tail -1; done
