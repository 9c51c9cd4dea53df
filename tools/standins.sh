# single-GPU multi-rank stand-ins of the N>1 bench path (gloo, several ranks on one GPU via HV_DEVICE_MAP)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4f_build.log 2>&1
HV_DEVICE_MAP=0,0 HV_BENCH_QWEN_LAYERS=8 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 --phi-layers 4 > gpurun_out/r4f_2ranks.json 2> gpurun_out/r4f_2ranks.err; echo "2ranks rc=$?"; tail -3 gpurun_out/r4f_2ranks.err | cut -c1-300
HV_DEVICE_MAP=0,0,0,0,0,0,0,0 HV_BENCH_QWEN_LAYERS=2 HV_CHURN_SECONDS=1.0 timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 8 --dist-backend gloo --steps 3 --warmup 3 --phi-layers 1 --no-kv > gpurun_out/r4f_8ranks.json 2> gpurun_out/r4f_8ranks.err; echo "8ranks rc=$?"; grep -iE "error|Traceback" gpurun_out/r4f_8ranks.err | head -5
