mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/gpu/r110_kvg4.py > gpurun_out/r110.json 2> gpurun_out/r110.err; echo rc=$?; tail -3 gpurun_out/r110.err
