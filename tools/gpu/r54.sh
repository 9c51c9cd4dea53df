set -x
mkdir -p gpurun_out
for v in kt128_s4 kt64_s4 kt64_s6 kt32_s8; do HARVEST_B200_LIB=build/ffnvar/lib_$v.so timeout 300 python tools/fused_probe.py hbm > gpurun_out/r54_$v.json 2> gpurun_out/r54_$v.err; echo $v rc=$?; done
