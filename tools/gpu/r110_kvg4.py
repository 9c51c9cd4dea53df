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
Orig = torch.cuda.Event

def b2b(dec, n=5):
    dec.step(); torch.cuda.synchronize()
    e0, e1 = Orig(enable_timing=True), Orig(enable_timing=True)
    e0.record()
    for i in range(n):
        dec.step()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n

out = {}
for cap in (64, 148):
    r = {}
    r["untraced"] = b2b(KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap))
    r["traced"] = b2b(KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap, trace=True))
    torch.cuda.Event = lambda enable_timing=False, **kw: Orig(enable_timing=True, **kw)
    r["untraced_timing_events"] = b2b(KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap))
    torch.cuda.Event = lambda enable_timing=False, **kw: Orig(enable_timing=False, **kw)
    r["traced_no_timing_events"] = b2b(KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap, trace=True)) if False else None
    torch.cuda.Event = Orig
    r["untraced_again"] = b2b(KVAttentionDecoder(kv, [0], q_heads=32, seed=1, max_ctas=cap))
    out[cap] = r
print(json.dumps(out, indent=1))
