set -x
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/r4_smoke.log 2>&1; tail -2 gpurun_out/r4_smoke.log
timeout 300 python -m pytest tests -q -m gpu > gpurun_out/r4_tests.log 2>&1; tail -3 gpurun_out/r4_tests.log
timeout 400 python tools/fetch_microbench.py > gpurun_out/r4_micro.json 2> gpurun_out/r4_micro.err; tail -3 gpurun_out/r4_micro.err
HV_DEVICE_MAP=0,0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/r4_bench2.json 2> gpurun_out/r4_bench2.err; tail -5 gpurun_out/r4_bench2.err; cat gpurun_out/r4_bench2.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r4_bench_ncu.log 2>&1; tail -2 gpurun_out/r4_bench_ncu.log
for w in host hbm kv; do timeout 300 ncu --set full --clock-control none --import-source on -k regex:copy -c 2 -o gpurun_out/r4_prof_$w -f python tools/profile_target.py $w ldg 2 > gpurun_out/r4_prof_$w.log 2>&1; tail -1 gpurun_out/r4_prof_$w.log; done
ls -la gpurun_out
