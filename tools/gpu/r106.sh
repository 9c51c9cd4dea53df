set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r106_smoke.log 2>&1; tail -1 gpurun_out/r106_smoke.log
timeout 1200 python bench.py > gpurun_out/r106_bench.json 2> gpurun_out/r106_bench.err; echo rc=$?; tail -3 gpurun_out/r106_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r106_ref.json 2> gpurun_out/r106_ref.err; echo rc=$?
