set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_kv_decode.py tests/test_gpu_churn.py -q -m gpu -x > gpurun_out/r80_t.log 2>&1; tail -25 gpurun_out/r80_t.log
HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0,0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 4 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --no-phi > gpurun_out/r80_bench4.json 2> gpurun_out/r80_bench4.err; echo rc=$?; tail -3 gpurun_out/r80_bench4.err
timeout 1200 python bench.py --no-cpu-baseline --no-kv > gpurun_out/r80_bench.json 2> gpurun_out/r80_bench.err; echo rc=$?; tail -3 gpurun_out/r80_bench.err
