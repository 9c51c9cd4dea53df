set -x
mkdir -p gpurun_out
HV_BENCH_QWEN_LAYERS=2 HV_DEVICE_MAP=0,0 timeout 2400 compute-sanitizer --target-processes all --tool memcheck --leak-check no --error-exitcode 9 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 1 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --no-phi --no-host-compare > gpurun_out/r92_mc2.json 2> gpurun_out/r92_mc2.err; echo "memcheck 2-rank rc=$?"; grep -E "ERROR SUMMARY|Invalid" gpurun_out/r92_mc2.err | sort | uniq -c | head
