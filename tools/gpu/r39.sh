set -x
timeout 600 python tools/kv_blocks_probe.py > gpurun_out/r39_kvprobe.json 2> gpurun_out/r39_kvprobe.err; tail -2 gpurun_out/r39_kvprobe.err
