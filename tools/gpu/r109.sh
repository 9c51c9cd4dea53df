mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/gpu/r109_kvg3.py > gpurun_out/r109.json 2> gpurun_out/r109.err; echo rc=$?; tail -3 gpurun_out/r109.err
