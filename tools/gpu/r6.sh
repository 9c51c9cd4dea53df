set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests -q -m gpu > gpurun_out/r6_tests.log 2>&1; tail -15 gpurun_out/r6_tests.log
timeout 600 python bench.py > gpurun_out/r6_bench.json 2> gpurun_out/r6_bench.err; tail -3 gpurun_out/r6_bench.err; cat gpurun_out/r6_bench.json
timeout 300 python bench.py --impl reference > gpurun_out/r6_ref.json 2> gpurun_out/r6_ref.err; tail -3 gpurun_out/r6_ref.err; cat gpurun_out/r6_ref.json
HV_DEVICE_MAP=0,0,0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 3 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/r6_bench3.json 2> gpurun_out/r6_bench3.err; tail -3 gpurun_out/r6_bench3.err; cat gpurun_out/r6_bench3.json
