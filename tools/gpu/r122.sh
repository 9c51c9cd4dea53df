mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_decode.py 2>&1 | tail -15
