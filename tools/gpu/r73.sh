set -x
mkdir -p gpurun_out
for v in 2 3 4; do HARVEST_B200_LIB=build/attnvar/lib_m$v.so timeout 300 python tools/attn_probe.py > gpurun_out/r73_m$v.json 2>gpurun_out/r73_m$v.err; echo m$v rc=$?; done
