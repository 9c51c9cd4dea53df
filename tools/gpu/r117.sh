mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest -q -m gpu tests 2>&1 | tail -4
