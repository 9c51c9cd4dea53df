set -x
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_churn.py -q -m gpu > gpurun_out/r20_tests.log 2>&1; tail -3 gpurun_out/r20_tests.log
HV_DEVICE_MAP=0,0 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --phi-layers 8 --no-kv > gpurun_out/r20_bench2.json 2> gpurun_out/r20_bench2.err; tail -5 gpurun_out/r20_bench2.err
