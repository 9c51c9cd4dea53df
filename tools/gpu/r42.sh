set -x
timeout 900 python bench.py --no-cpu-baseline --no-kv --no-host-compare > gpurun_out/r42_bench.json 2> gpurun_out/r42_bench.err; echo rc=$?
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --no-phi --no-host-compare > gpurun_out/r42_bench2.json 2> gpurun_out/r42_bench2.err; echo rc=$?
