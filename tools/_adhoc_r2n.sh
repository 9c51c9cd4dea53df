bash tools/gpu_suite.sh r2n build
timeout 900 ncu --set full --clock-control none --import-source on -k regex:desc_op_kernel -c 1 -o gpurun_out/r2n_checked16 -f python tools/profile_target.py checked ldg16 2 > gpurun_out/r2n_ncu1.log 2>&1; echo ncu16 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:desc_op_kernel -c 1 -o gpurun_out/r2n_checked8 -f python tools/profile_target.py checked ldg 2 > gpurun_out/r2n_ncu2.log 2>&1; echo ncu8 rc=$?
