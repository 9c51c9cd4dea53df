set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x > gpurun_out/r72_t.log 2>&1; tail -25 gpurun_out/r72_t.log
timeout 300 python tools/attn_probe.py > gpurun_out/r72_attn.json 2>gpurun_out/r72_attn.err; echo rc=$?
