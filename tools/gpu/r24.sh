set -x
HV_BENCH_QWEN_LAYERS=2 HV_DEVICE_MAP=0,0,0,0,0,0,0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 8 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --phi-layers 2 > gpurun_out/r24_bench8.json 2> gpurun_out/r24_bench8.err; echo rc=$?; tail -15 gpurun_out/r24_bench8.err; cat gpurun_out/r24_bench8.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r24_ref.json 2>&1; tail -2 gpurun_out/r24_ref.json
