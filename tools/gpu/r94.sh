set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.used --format=csv
HV_CHURN_SECONDS=20 HV_BENCH_QWEN_LAYERS=2 timeout 1500 python bench.py --no-cpu-baseline --no-kv --steps 3 > gpurun_out/r94_soak1.json 2> gpurun_out/r94_soak1.err; echo rc=$?; tail -3 gpurun_out/r94_soak1.err
HV_CHURN_SECONDS=20 HV_BENCH_QWEN_LAYERS=2 HV_DEVICE_MAP=0,0,0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 4 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --no-phi > gpurun_out/r94_soak4.json 2> gpurun_out/r94_soak4.err; echo rc=$?; tail -3 gpurun_out/r94_soak4.err
