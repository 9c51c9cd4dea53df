bash tools/gpu_suite.sh r2e build file:tests/test_gpu_ipc.py,tests/test_gpu_decode.py
python tools/fused_probe.py hbm > gpurun_out/r2e_fused_tma.json 2>&1; echo tma rc=$?
HARVEST_B200_LIB=build/ffn_cpasync/libharvest_b200.so python tools/fused_probe.py hbm > gpurun_out/r2e_fused_cpasync.json 2>&1; echo cpasync rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/nccl_rankgroup_smoke.py --same-gpu > gpurun_out/r2e_nccl_same_gpu.log 2>&1; echo nccl rc=$?; tail -3 gpurun_out/r2e_nccl_same_gpu.log
