mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_kv_decode.py tests/test_gpu_kv.py 2>&1 | tail -1
timeout 600 python tools/kv_decode_probe.py > gpurun_out/r125_kvdp.json 2> gpurun_out/r125_kvdp.err; echo rc=$?; tail -2 gpurun_out/r125_kvdp.err
