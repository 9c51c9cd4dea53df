bash tools/gpu_suite.sh r2z build
python tools/fused_probe.py hbm > gpurun_out/r2z_fused_base.json 2>&1; echo base rc=$?
for v in ffn_sd4 ffn_sd5 ffn_s4; do HARVEST_B200_LIB=build/$v/libharvest_b200.so python tools/fused_probe.py hbm > gpurun_out/r2z_fused_$v.json 2>&1; echo $v rc=$?; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expert_ffn -c 2 -o gpurun_out/r2z_ffn -f python tools/profile_target.py fused ldg 1 > gpurun_out/r2z_ncu.log 2>&1; echo ncu rc=$?
