set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --no-cpu-baseline --no-kv > gpurun_out/r95_bench.json 2> gpurun_out/r95_bench.err; echo rc=$?; tail -3 gpurun_out/r95_bench.err
HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0,0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 4 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --no-phi > gpurun_out/r95_bench4.json 2> gpurun_out/r95_bench4.err; echo rc=$?; tail -3 gpurun_out/r95_bench4.err
