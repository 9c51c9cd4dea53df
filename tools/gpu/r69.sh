set -x
mkdir -p gpurun_out
for v in 0 2 3; do HARVEST_B200_LIB=build/attnvar/lib_h$v.so timeout 300 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x > gpurun_out/r69_t$v.log 2>&1; tail -1 gpurun_out/r69_t$v.log; HARVEST_B200_LIB=build/attnvar/lib_h$v.so timeout 300 python tools/attn_probe.py > gpurun_out/r69_h$v.json 2>gpurun_out/r69_h$v.err; echo h$v rc=$?; done
