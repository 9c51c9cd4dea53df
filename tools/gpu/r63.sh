set -x
mkdir -p gpurun_out
timeout 300 python tools/kv_decode_repro.py > gpurun_out/r63_repro.log 2>&1; echo rc=$?; tail -3 gpurun_out/r63_repro.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/kv_decode_repro.py 2 1024 > gpurun_out/r63_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -A12 "Invalid\|ERROR SUMMARY" gpurun_out/r63_memcheck.log | head -40
HV_BENCH_QWEN_LAYERS=2 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-phi --no-churn --no-host-compare > gpurun_out/r63_bench2.json 2> gpurun_out/r63_bench2.err; echo rc=$?
grep -v CUDAEvent gpurun_out/r63_bench2.err | grep "rank0\]" | head -30
