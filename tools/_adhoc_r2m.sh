bash tools/gpu_suite.sh r2m build
timeout 900 ncu --set full --clock-control none --import-source on -k regex:CopyDigest -c 1 -o gpurun_out/r2m_checked16 -f python tools/profile_target.py checked ldg16 2 > gpurun_out/r2m_ncu1.log 2>&1; echo ncu16 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:CopyDigest -c 1 -o gpurun_out/r2m_checked8 -f python tools/profile_target.py checked ldg 2 > gpurun_out/r2m_ncu2.log 2>&1; echo ncu8 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:desc_op_kernel -c 1 -o gpurun_out/r2m_copy16 -f python tools/profile_target.py hbm ldg16 2 > gpurun_out/r2m_ncu3.log 2>&1; echo ncucopy rc=$?
