set -x
timeout 600 python bench.py --impl reference > gpurun_out/r40_ref.json 2> gpurun_out/r40_ref.err; echo rc=$?
timeout 1200 python bench.py > gpurun_out/r40_bench.json 2> gpurun_out/r40_bench.err; echo rc=$?
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --phi-layers 8 > gpurun_out/r40_bench2.json 2> gpurun_out/r40_bench2.err; echo rc=$?
