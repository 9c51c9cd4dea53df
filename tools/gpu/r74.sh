set -x
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x -k "kernel_matches and 128" > gpurun_out/r74_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/r74_racecheck.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x > gpurun_out/r74_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/r74_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x -k "kernel_matches and 128" > gpurun_out/r74_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -2 gpurun_out/r74_synccheck.log
timeout 1200 python bench.py > gpurun_out/r74_bench.json 2> gpurun_out/r74_bench.err; echo rc=$?; tail -3 gpurun_out/r74_bench.err
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --phi-layers 4 > gpurun_out/r74_bench2.json 2> gpurun_out/r74_bench2.err; echo rc=$?; tail -3 gpurun_out/r74_bench2.err
