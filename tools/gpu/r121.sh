mkdir -p gpurun_out
for v in head old v0 head; do HARVEST_B200_LIB=build/ffnvar3/$v.so timeout 300 python tools/fused_probe.py hbm > gpurun_out/r121_$v.json 2> gpurun_out/r121_$v.err; echo $v rc=$?; tail -2 gpurun_out/r121_$v.err; python -c "
import json
d=json.load(open('gpurun_out/r121_$v.json'))
print('$v', {k: (round(r['fused_down']['weight_GBps']), round(r['fused_gate_up']['weight_GBps']), round(r['fused']['weight_GBps'])) for k,r in d.items()})"; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv
