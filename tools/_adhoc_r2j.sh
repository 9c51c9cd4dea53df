bash tools/gpu_suite.sh r2j build smoke tests
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; echo bench rc=$?; tail -2 gpurun_out/r2j_bench.err | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2j_ref.json 2> gpurun_out/r2j_ref.err; echo ref rc=$?
