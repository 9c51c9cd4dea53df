#!/bin/bash
# NVLink evidence for the peer-fetch kernels (needs a box with >= 2 GPUs):
# per-launch NVLink receive/transmit bytes, DRAM traffic and duration of K2
# (a Qwen stage of 53 x 17.3 MB experts) and K1 (config 1's 1,024 x 64 KiB
# pages) reading a VMM pool on cuda:1 from cuda:0.  Usage:
#   bash tools/ncu_nvlink.sh TAG [engine]
# Output: gpurun_out/TAG_nvlink_{peer,peer_kv}.csv; nvlrx__bytes.sum on the
# reading GPU should equal the algorithmic bytes (917 MB / 64 MiB per launch).
TAG=${1:-nvl}; ENG=${2:-ldg}
mkdir -p gpurun_out
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for MODE in peer peer_kv; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:"copy" --csv \
    --log-file gpurun_out/${TAG}_nvlink_${MODE}.csv python tools/profile_target.py $MODE $ENG 3 \
    > gpurun_out/${TAG}_nvlink_${MODE}.log 2>&1
  echo "$MODE rc=$?"
done
