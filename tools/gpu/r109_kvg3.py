import json, sys, time
import torch
sys.path.insert(0, ".")
from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager
from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
from paper_2602_00328_b200.runtime import Durability
from paper_2602_00328_b200.system import HarvestSystem
m = LLAMA3_8B
ctx = 131072
nblk = ctx // m.block_tokens
sysm = HarvestSystem(0, donors=[0], donor_bytes=(nblk // 64 + 2) * 64 * m.block_bytes, host_bytes=1, local_bytes=1)
kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=1, slab_blocks=64, durability=Durability.LOSSY, content="fp16")
kv.append_kv(0, ctx)
kv.evict(nblk * m.block_bytes)
out = {}
for cap in (64, 148):
    r = {}
    # A: back to back with trace, report of the last step
    dec = KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap, trace=True)
    dec.step(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(5):
        dec.step()
    e1.record(); e1.synchronize()
    r["b2b_traced_ms"] = e0.elapsed_time(e1) / 5
    r["b2b_traced_last"] = {k: round(v, 3) for k, v in dec.overlap_report().items()}
    # B: synchronize after each step
    dec2 = KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap)
    dec2.step(); torch.cuda.synchronize()
    ws = []
    for i in range(5):
        t0 = time.perf_counter(); dec2.step(); torch.cuda.synchronize(); ws.append((time.perf_counter() - t0) * 1e3)
    r["synced_wall_ms"] = ws
    # C: back to back, host sleeps 10 ms after each enqueue (host far slower than device)
    e0.record()
    for i in range(5):
        dec2.step(); time.sleep(0.02)
    e1.record(); e1.synchronize()
    r["b2b_sleep20_ms"] = e0.elapsed_time(e1) / 5
    # D: profile kernel durations of 2 b2b steps
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for i in range(2):
            dec2.step()
        torch.cuda.synchronize()
    ev = [(e.key, e.device_time_total / 1e3, e.count) for e in p.key_averages()]
    r["kernels"] = sorted([(n[:60], round(t, 3), c) for n, t, c in ev if t > 0], key=lambda x: -x[1])[:10]
    out[cap] = r
print(json.dumps(out, indent=1))
