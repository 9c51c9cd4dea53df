set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r124_smoke.log 2>&1; tail -1 gpurun_out/r124_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r124_tests.log 2>&1; tail -2 gpurun_out/r124_tests.log
timeout 1200 python bench.py > gpurun_out/r124_bench.json 2> gpurun_out/r124_bench.err; echo rc=$?; tail -3 gpurun_out/r124_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r124_ref.json 2> gpurun_out/r124_ref.err; echo rc=$?
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29545 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --phi-layers 4 > gpurun_out/r124_bench2.json 2> gpurun_out/r124_bench2.err; echo rc=$?; tail -3 gpurun_out/r124_bench2.err
HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0,0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29546 bench.py --gpus 4 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --phi-layers 2 > gpurun_out/r124_bench4.json 2> gpurun_out/r124_bench4.err; echo rc=$?; tail -3 gpurun_out/r124_bench4.err
