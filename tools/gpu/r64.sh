set -x
mkdir -p gpurun_out
for i in 1 2; do HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-phi --no-churn > gpurun_out/r64_bench2_$i.json 2> gpurun_out/r64_bench2_$i.err; echo rc=$?; grep -v CUDAEvent gpurun_out/r64_bench2_$i.err | grep "rank0\]" | grep -v "\^\^" | head -12; done
