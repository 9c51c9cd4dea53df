set -x
timeout 600 python -m pytest tests/test_gpu_kv.py tests/test_gpu_vllm_adapter.py -q -m gpu > gpurun_out/r30_tests.log 2>&1; tail -2 gpurun_out/r30_tests.log
HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-phi --no-churn > gpurun_out/r30_bench2.json 2> gpurun_out/r30_bench2.err; echo rc=$?; tail -3 gpurun_out/r30_bench2.err
