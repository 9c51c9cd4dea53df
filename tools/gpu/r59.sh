set -x
mkdir -p gpurun_out
python -c "
import sys; sys.path.insert(0,'tools')
import nvlink_counters as n
c=n.NvlinkCounters(0); print('nvlink', c.snapshot(), c.error)" > gpurun_out/r59_nvl.log 2>&1; cat gpurun_out/r59_nvl.log
timeout 1200 python bench.py > gpurun_out/r59_bench.json 2> gpurun_out/r59_bench.err; echo rc=$?; tail -3 gpurun_out/r59_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r59_ref.json 2> gpurun_out/r59_ref.err; echo rc=$?
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --phi-layers 4 > gpurun_out/r59_bench2.json 2> gpurun_out/r59_bench2.err; echo rc=$?; tail -3 gpurun_out/r59_bench2.err
