bash tools/gpu_suite.sh r2v build file:tests/test_gpu_kv_decode.py
python tools/kv_decode_probe.py > gpurun_out/r2v_kvdec.json 2>&1; echo pdl rc=$?
