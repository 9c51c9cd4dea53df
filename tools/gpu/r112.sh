mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/event_probe.py > gpurun_out/r112_carve1.json 2> gpurun_out/r112_carve1.err; echo rc=$?; tail -2 gpurun_out/r112_carve1.err
HARVEST_B200_LIB=build/carve0/lib.so timeout 600 python tools/event_probe.py > gpurun_out/r112_carve0.json 2> gpurun_out/r112_carve0.err; echo rc=$?; tail -2 gpurun_out/r112_carve0.err
timeout 600 python tools/kv_decode_probe.py > gpurun_out/r112_kvdp.json 2> gpurun_out/r112_kvdp.err; echo rc=$?; tail -2 gpurun_out/r112_kvdp.err
