mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/gather_order_probe.py > gpurun_out/r114.json 2> gpurun_out/r114.err; echo rc=$?; tail -3 gpurun_out/r114.err
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_kv_decode.py 2>&1 | tail -2
