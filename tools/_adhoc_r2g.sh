bash tools/gpu_suite.sh r2g build smoke tests
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo bench rc=$?; tail -2 gpurun_out/r2g_bench.err | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2g_ref.json 2> gpurun_out/r2g_ref.err; echo ref rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:desc_op_kernel -c 1 -o gpurun_out/r2g_check -f python tools/profile_target.py check > gpurun_out/r2g_ncu_check.log 2>&1; echo ncu rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 2 --warmup 3 --no-kv --no-churn --no-sweep --no-cpu-baseline > gpurun_out/r2g_launches.log 2>&1; echo launches rc=$?
HARVEST_B200_LIB=build/attn_w4/libharvest_b200.so python tools/attn_probe.py > gpurun_out/r2g_attn_w4.json 2>&1; echo w4 rc=$?
