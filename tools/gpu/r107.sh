set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for w in 4 8; do HARVEST_B200_LIB=build/attnvar2/lib_w$w.so timeout 400 python tools/kv_gather_probe.py > gpurun_out/r107_w$w.json 2> gpurun_out/r107_w$w.err; echo w$w rc=$?; tail -2 gpurun_out/r107_w$w.err; done
