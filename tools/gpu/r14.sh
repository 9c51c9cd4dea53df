set -x
timeout 600 python -m pytest tests/test_gpu_kv.py -q -m gpu > gpurun_out/r14_tests.log 2>&1; tail -3 gpurun_out/r14_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r14_bench.json 2> gpurun_out/r14_bench.err; tail -5 gpurun_out/r14_bench.err; cat gpurun_out/r14_bench.json
HV_DEVICE_MAP=0,0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-host-compare > gpurun_out/r14_bench2.json 2> gpurun_out/r14_bench2.err; tail -5 gpurun_out/r14_bench2.err; cat gpurun_out/r14_bench2.json
