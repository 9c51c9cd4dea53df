set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_kv_decode.py -q -m gpu -x > gpurun_out/r101_t.log 2>&1; tail -2 gpurun_out/r101_t.log
timeout 1500 python bench.py --no-cpu-baseline --no-churn > gpurun_out/r101_bench.json 2> gpurun_out/r101_bench.err; echo rc=$?; tail -3 gpurun_out/r101_bench.err
HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --phi-layers 2 > gpurun_out/r101_bench2.json 2> gpurun_out/r101_bench2.err; echo rc=$?; tail -3 gpurun_out/r101_bench2.err
