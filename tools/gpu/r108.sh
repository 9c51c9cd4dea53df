mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/gpu/r108_kvg2.py > gpurun_out/r108.json 2> gpurun_out/r108.err; echo rc=$?; tail -3 gpurun_out/r108.err
