import json, os, sys, time
import torch
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager
from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
from paper_2602_00328_b200.runtime import Durability
from paper_2602_00328_b200.system import HarvestSystem
m = LLAMA3_8B
batch, ctx = 1, 131072
nblk = batch * ctx // m.block_tokens
sysm = HarvestSystem(0, donors=[0], donor_bytes=(nblk // 64 + 2) * 64 * m.block_bytes, host_bytes=1, local_bytes=1)
kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=1, slab_blocks=64, durability=Durability.LOSSY, content="fp16")
kv.append_kv(0, ctx)
kv.evict(nblk * m.block_bytes)
out = {}
for cap in (64, 148):
    dec = KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap, trace=True)
    rows = []
    for i in range(6):
        t0 = time.perf_counter()
        dec.step()
        t1 = time.perf_counter()
        rep = dec.overlap_report()   # syncs
        t2 = time.perf_counter()
        rows.append({"host_enqueue_ms": (t1 - t0) * 1e3, "wall_to_done_ms": (t2 - t0) * 1e3, **{k: round(v, 3) for k, v in rep.items()}})
    # back to back, untraced, event timed, and host enqueue times
    dec2 = KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap)
    dec2.step(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hs = []
    e0.record()
    for i in range(5):
        t0 = time.perf_counter(); dec2.step(); hs.append((time.perf_counter() - t0) * 1e3)
    e1.record(); e1.synchronize()
    out[cap] = {"traced_steps": rows, "b2b_ms_per_step": e0.elapsed_time(e1) / 5, "b2b_host_ms": hs}
print(json.dumps(out, indent=1))
