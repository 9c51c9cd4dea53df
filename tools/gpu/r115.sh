mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python tools/moe_order_probe.py > gpurun_out/r115.json 2> gpurun_out/r115.err; echo rc=$?; tail -3 gpurun_out/r115.err
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_decode.py 2>&1 | tail -2
