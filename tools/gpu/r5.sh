set -x
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/r5_smoke.log 2>&1; tail -2 gpurun_out/r5_smoke.log
timeout 400 python -m pytest tests -q -m gpu -x > gpurun_out/r5_tests.log 2>&1; tail -15 gpurun_out/r5_tests.log
timeout 400 python tools/fetch_microbench.py > gpurun_out/r5_micro.json 2> gpurun_out/r5_micro.err; tail -3 gpurun_out/r5_micro.err
for w in host hbm; do timeout 300 ncu --set full --clock-control none --import-source on -k regex:desc_op_kernel -c 2 -o gpurun_out/r5_prof_$w -f python tools/profile_target.py $w ldg 2 > gpurun_out/r5_prof_$w.log 2>&1; tail -1 gpurun_out/r5_prof_$w.log; done
