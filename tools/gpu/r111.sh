mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/event_probe.py > gpurun_out/r111.json 2> gpurun_out/r111.err; echo rc=$?; tail -3 gpurun_out/r111.err
