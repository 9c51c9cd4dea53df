set -x
mkdir -p gpurun_out
for v in kt64_s4_p0 kt64_s4_p1 kt64_s3_p1 kt128_s3_p1; do HARVEST_B200_LIB=build/ffnvar/lib_$v.so timeout 300 python -m pytest tests/test_gpu_decode.py -q -m gpu -x -k "fused" > gpurun_out/r57_t_$v.log 2>&1; tail -1 gpurun_out/r57_t_$v.log; HARVEST_B200_LIB=build/ffnvar/lib_$v.so timeout 300 python tools/fused_probe.py hbm > gpurun_out/r57_$v.json 2> gpurun_out/r57_$v.err; echo $v rc=$?; done
