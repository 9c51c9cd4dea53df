bash tools/gpu_suite.sh r3b build file:tests/test_gpu_decode.py
python tools/fused_probe.py hbm > gpurun_out/r3b_fused_pdl.json 2>&1; echo pdl rc=$?
python tools/fused_probe.py hbm --no-pdl > gpurun_out/r3b_fused_nopdl.json 2>&1; echo nopdl rc=$?
