set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kv.py -q -m gpu > gpurun_out/r50_tests.log 2>&1; tail -3 gpurun_out/r50_tests.log
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-phi --no-churn --no-host-compare > gpurun_out/r50_bench2.json 2> gpurun_out/r50_bench2.err; echo rc=$?; tail -3 gpurun_out/r50_bench2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r50_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r50_bench_ncu.log 2>&1; echo rc=$?; tail -2 gpurun_out/r50_bench_ncu.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"desc_op" -c 2 -o gpurun_out/r50_prof_host_ldg256 -f python tools/profile_target.py host ldg256 2 > gpurun_out/r50_prof.log 2>&1; echo rc=$?; tail -2 gpurun_out/r50_prof.log
