set -x
HV_DEVICE_MAP=0,0 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --phi-layers 8 > gpurun_out/r19_bench2.json 2> gpurun_out/r19_bench2.err; tail -5 gpurun_out/r19_bench2.err; cat gpurun_out/r19_bench2.json
