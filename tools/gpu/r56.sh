set -x
mkdir -p gpurun_out
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --no-churn --phi-layers 4 > gpurun_out/r56_bench2.json 2> gpurun_out/r56_bench2.err; echo rc=$?; tail -3 gpurun_out/r56_bench2.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"expert_ffn" -c 2 -o gpurun_out/r56_prof_fused -f python tools/profile_target.py fused x 1 > gpurun_out/r56_prof.log 2>&1; echo rc=$?; tail -2 gpurun_out/r56_prof.log
