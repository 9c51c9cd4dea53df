set -x
mkdir -p gpurun_out
HV_BENCH_QWEN_LAYERS=2 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --no-churn --phi-layers 4 > gpurun_out/r93_bench2.json 2> gpurun_out/r93_bench2.err; echo rc=$?; tail -3 gpurun_out/r93_bench2.err
