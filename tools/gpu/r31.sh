set -x
timeout 900 python bench.py > gpurun_out/r31_bench.json 2> gpurun_out/r31_bench.err; echo rc=$?; tail -3 gpurun_out/r31_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r31_ref.json 2> gpurun_out/r31_ref.err; echo rc=$?; tail -2 gpurun_out/r31_ref.err
HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --phi-layers 2 > gpurun_out/r31_bench2.json 2> gpurun_out/r31_bench2.err; echo rc=$?; tail -3 gpurun_out/r31_bench2.err
