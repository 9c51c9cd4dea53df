mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_kv_decode.py tests/test_gpu_kv.py tests/test_gpu_vllm_adapter.py 2>&1 | tail -2
timeout 600 python tools/kv_decode_probe.py > gpurun_out/r116_kvdp.json 2> gpurun_out/r116_kvdp.err; echo rc=$?; tail -2 gpurun_out/r116_kvdp.err
timeout 600 python tools/gpu/r108_kvg2.py > gpurun_out/r116_host.json 2> gpurun_out/r116_host.err; echo rc=$?
