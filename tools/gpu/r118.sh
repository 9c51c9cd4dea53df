set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r118_smoke.log 2>&1; tail -1 gpurun_out/r118_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r118_tests.log 2>&1; tail -2 gpurun_out/r118_tests.log
timeout 1200 python bench.py > gpurun_out/r118_bench.json 2> gpurun_out/r118_bench.err; echo rc=$?; tail -3 gpurun_out/r118_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r118_ref.json 2> gpurun_out/r118_ref.err; echo rc=$?
HV_BENCH_QWEN_LAYERS=8 HV_DEVICE_MAP=0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --phi-layers 4 > gpurun_out/r118_bench2.json 2> gpurun_out/r118_bench2.err; echo rc=$?; tail -3 gpurun_out/r118_bench2.err
HV_BENCH_QWEN_LAYERS=4 HV_DEVICE_MAP=0,0,0,0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29536 bench.py --gpus 4 --steps 3 --warmup 3 --dist-backend gloo --no-cpu-baseline --no-kv --phi-layers 2 > gpurun_out/r118_bench4.json 2> gpurun_out/r118_bench4.err; echo rc=$?; tail -3 gpurun_out/r118_bench4.err
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x -k "kernel_matches and 128" > gpurun_out/r118_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/r118_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x -k "kernel_matches and 128" > gpurun_out/r118_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -2 gpurun_out/r118_synccheck.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_kv_decode.py -q -m gpu -x > gpurun_out/r118_memcheck_kvdec.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/r118_memcheck_kvdec.log
