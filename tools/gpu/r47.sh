set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r47_tests.log 2>&1; tail -3 gpurun_out/r47_tests.log
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0,0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 4 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --no-phi --no-churn --no-host-compare > gpurun_out/r47_bench4.json 2> gpurun_out/r47_bench4.err; echo rc=$?
