set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kv_decode.py tests/test_gpu_kv.py tests/test_gpu_vllm_adapter.py -q -m gpu -x > gpurun_out/r65_tests.log 2>&1; tail -2 gpurun_out/r65_tests.log
for i in 1 2 3; do HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-phi --no-churn > gpurun_out/r65_bench2_$i.json 2> gpurun_out/r65_bench2_$i.err; echo rc=$?; done
