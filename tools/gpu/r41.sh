set -x
for eng in tma ldg16; do timeout 300 ncu --set full --clock-control none --import-source on -k regex:"block_copy" -c 2 -o gpurun_out/r41_prof_blocks_$eng -f python tools/profile_target.py blocks $eng 2 > gpurun_out/r41_prof_blocks_$eng.log 2>&1; tail -1 gpurun_out/r41_prof_blocks_$eng.log; done
