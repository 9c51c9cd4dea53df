set -x
mkdir -p gpurun_out
for v in 3 4 6 8; do HARVEST_B200_LIB=build/ffnvar2/lib_d$v.so timeout 300 python tools/fused_probe.py hbm > gpurun_out/r86_d$v.json 2> gpurun_out/r86_d$v.err; echo d$v rc=$?; done
HARVEST_B200_LIB=build/ffnvar2/lib_d6.so timeout 300 python -m pytest tests/test_gpu_decode.py -q -m gpu -x -k fused 2>&1 | tail -1
