mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r126_smoke.log 2>&1; tail -1 gpurun_out/r126_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r126_tests.log 2>&1; tail -2 gpurun_out/r126_tests.log | head -1
timeout 1200 python bench.py > gpurun_out/r126_bench.json 2> gpurun_out/r126_bench.err; echo rc=$?; tail -3 gpurun_out/r126_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r126_ref.json 2> gpurun_out/r126_ref.err; echo ref rc=$?
