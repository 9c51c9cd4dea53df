# final round-2 validation: tests, the contract bench and reference lines, the
# launch list of the bench command, and ncu captures of the step's kernels
TAG=${1:-r3f}
bash tools/gpu_suite.sh $TAG build smoke tests
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?; tail -2 gpurun_out/${TAG}_bench.err | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-kv --no-churn --no-sweep --no-cpu-baseline > gpurun_out/${TAG}_launches.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:desc_digest_tma -c 1 -o gpurun_out/${TAG}_check -f python tools/profile_target.py check > gpurun_out/${TAG}_ncu_check.log 2>&1; echo ncu check rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_decode -c 1 -o gpurun_out/${TAG}_attn -f python tools/profile_target.py attn ldg 1 > gpurun_out/${TAG}_ncu_attn.log 2>&1; echo ncu attn rc=$?
