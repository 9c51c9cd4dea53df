set -x
mkdir -p gpurun_out/r91
for t in host_overhead graph_probe il_probe kv_blocks_probe vmm_probe wc_probe ffn_probe kv_decode_repro; do timeout 300 python tools/$t.py > gpurun_out/r91/$t.out 2> gpurun_out/r91/$t.err; echo "$t rc=$?"; done
for spec in "host ldg" "hbm tma" "kv ldg" "blocks tma" "fused x"; do set -- $spec; timeout 120 python tools/profile_target.py $1 $2 1 > gpurun_out/r91/pt_$1.out 2>&1; echo "profile_target $1 rc=$?"; done
timeout 600 python tools/fetch_microbench.py > gpurun_out/r91/fetch_microbench.out 2> gpurun_out/r91/fetch_microbench.err; echo "fetch_microbench rc=$?"
