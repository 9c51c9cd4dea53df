"""KV decode gather mode (K1 per layer on the fetch stream, K5 on the compute
stream) over a self-donor VMM pool: step time and the device-clock gather /
attention sums for several K1 grid caps, against the in-place mode.  Says
whether K1 and K5 overlap (span < serial) and which one bounds the step.
Prints JSON."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kv_decode_probe import timed  # noqa: E402
from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager  # noqa: E402
from paper_2602_00328_b200.kv_decode import KVAttentionDecoder  # noqa: E402
from paper_2602_00328_b200.runtime import Durability  # noqa: E402
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402


def case(batch, ctx, caps=(16, 32, 64, 148, 0)):
    m = LLAMA3_8B
    nblk = batch * ctx // m.block_tokens
    sysm = HarvestSystem(0, donors=[0], donor_bytes=(nblk // 64 + 2) * 64 * m.block_bytes, host_bytes=1,
                         local_bytes=1)
    kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=1, slab_blocks=64, durability=Durability.LOSSY,
                        content="fp16")
    for s in range(batch):
        kv.append_kv(s, ctx)
    kv.evict(nblk * m.block_bytes)
    seqs = list(range(batch))
    out = {}
    ref, ms = timed(KVAttentionDecoder(kv, seqs, q_heads=32, seed=1, fused=True))
    out["in_place"] = {"ms_per_step": ms}
    for cap in caps:
        dec = KVAttentionDecoder(kv, seqs, q_heads=32, seed=1, max_ctas=cap)
        o, ms = timed(dec)
        assert torch.equal(o, ref)
        tr = KVAttentionDecoder(kv, seqs, q_heads=32, seed=1, max_ctas=cap, trace=True)
        tr.step()
        rep = tr.overlap_report()
        out[f"gather_max_ctas_{cap}"] = {"ms_per_step": ms, **rep}
        del dec, tr
    sysm.loop.run()
    kv.close()
    sysm.close()
    return out


if __name__ == "__main__":
    print(json.dumps({"config1_4x4k": case(4, 4096), "context_128k": case(1, 131072)}, indent=1))
