set -x
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r13_bench.json 2> gpurun_out/r13_bench.err; tail -3 gpurun_out/r13_bench.err; cat gpurun_out/r13_bench.json
HV_DEVICE_MAP=0,0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-host-compare > gpurun_out/r13_bench2.json 2> gpurun_out/r13_bench2.err; tail -3 gpurun_out/r13_bench2.err; cat gpurun_out/r13_bench2.json
