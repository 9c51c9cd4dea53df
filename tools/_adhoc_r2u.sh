bash tools/gpu_suite.sh r2u build file:tests/test_gpu_kv_decode.py
python tools/kv_decode_probe.py > gpurun_out/r2u_kvdec_pdl.json 2>&1; echo pdl rc=$?
python tools/kv_decode_probe.py --no-overlap > gpurun_out/r2u_kvdec_nopdl.json 2>&1; echo nopdl rc=$?
