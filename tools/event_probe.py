"""Cross-stream pipelines (KV decode gather mode: K1 on the fetch stream, K5
on the compute stream; staged MoE decode: K2 fetch, cuBLAS compute) with the
stream-ordering events created with and without timing.  Self-donor VMM pool
(peer tier = this GPU's HBM).  Prints JSON: ms per step for each variant."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200.decode import MoEDecoder  # noqa: E402
from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager  # noqa: E402
from paper_2602_00328_b200.kv_decode import KVAttentionDecoder  # noqa: E402
from paper_2602_00328_b200.moe import (QWEN15_MOE_A27B, ExpertFetcher, ExpertResidency, ExpertStore,  # noqa: E402
                                       MoEProfile, rebalance)
from paper_2602_00328_b200.runtime import Durability  # noqa: E402
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402

Orig = torch.cuda.Event


def b2b(step, n=5):
    step()
    torch.cuda.synchronize()
    e0, e1 = Orig(enable_timing=True), Orig(enable_timing=True)
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


def variants(make):
    out = {}
    for name, timing in (("default_events", None), ("timing_events", True), ("no_timing_events", False)):
        if timing is not None:
            torch.cuda.Event = lambda enable_timing=False, _t=timing, **kw: Orig(enable_timing=_t, **kw)
        try:
            out[name] = b2b(make())
        finally:
            torch.cuda.Event = Orig
    return out


def kv_case(ctx, caps=(64, 148)):
    m = LLAMA3_8B
    nblk = ctx // m.block_tokens
    sysm = HarvestSystem(0, donors=[0], donor_bytes=(nblk // 64 + 2) * 64 * m.block_bytes, host_bytes=1,
                         local_bytes=1)
    kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=1, slab_blocks=64, durability=Durability.LOSSY,
                        content="fp16")
    kv.append_kv(0, ctx)
    kv.evict(nblk * m.block_bytes)
    out = {f"gather_max_ctas_{c}": variants(lambda c=c: KVAttentionDecoder(kv, [0], q_heads=32, seed=1,
                                                                            max_ctas=c).step)
           for c in caps}
    sysm.loop.run()
    kv.close()
    sysm.close()
    return out


def moe_case(layers=8, tokens=32):
    q = QWEN15_MOE_A27B
    model = MoEProfile(q.name, layers, q.num_experts, q.top_k, q.expert_size, hidden=q.hidden,
                       intermediate=q.intermediate)
    L, E, S = layers, q.num_experts, q.expert_size
    sysm = HarvestSystem(0, donors=[0], donor_bytes=L * E * S + (64 << 20), host_bytes=L * E * S, local_bytes=1 << 20)
    store = ExpertStore(model, sysm.host_id, sysm.host)
    store.fill_host(0, weights=True)
    res = ExpertResidency(model)
    rebalance(sysm.loop, sysm.runtime, model, res, np.ones((L, E), dtype=np.int64), sysm.host_id,
              max_migrations=L * E, store=store)
    sysm.loop.run()
    fetcher = ExpertFetcher(sysm.runtime, model, res, store)
    def stepper(**kw):
        dec = MoEDecoder(fetcher, tokens=tokens, seed=0, **kw)
        return lambda: dec.step(dec.x0)

    out = {}
    for mb in (1, 2):
        out[f"staged_mb{mb}"] = variants(lambda mb=mb: stepper(microbatches=mb))
    out["fused_mb2"] = variants(lambda: stepper(microbatches=2, fused=True))
    return out


if __name__ == "__main__":
    print(json.dumps({"kv_128k": kv_case(131072), "kv_4k": kv_case(4096 * 4), "moe_qwen_8l": moe_case()},
                     indent=1))
