"""KV decode gather mode: host issue order of the per-layer K1 / K5 pair and
the kind of stream events, eager and as a CUDA graph.  Self-donor VMM pool
(peer tier = this GPU's HBM), Llama-3-8B shapes.  Prints JSON: ms per step,
back-to-back steps; every variant's output is checked against the in-place
mode's."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from event_probe import b2b  # noqa: E402
from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager  # noqa: E402
from paper_2602_00328_b200.kv_decode import KVAttentionDecoder  # noqa: E402
from paper_2602_00328_b200.runtime import Durability  # noqa: E402
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402


def case(batch, ctx, cap=64):
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
    ref = KVAttentionDecoder(kv, seqs, q_heads=32, seed=1, fused=True)
    want = ref.step().clone()
    out = {"in_place": b2b(ref.step)}
    for ahead in (False, True):
        for timed in (False, True):
            for graph in (False, True):
                KVAttentionDecoder.issue_ahead, KVAttentionDecoder.timed_events = ahead, timed
                if graph and timed:
                    continue            # no events inside a graph
                dec = KVAttentionDecoder(kv, seqs, q_heads=32, seed=1, max_ctas=cap)
                if graph:
                    dec.capture_graph()
                assert torch.equal(dec.step(), want)
                out[f"ahead={int(ahead)} timed={int(timed)} graph={int(graph)}"] = b2b(dec.step)
                del dec
    KVAttentionDecoder.issue_ahead, KVAttentionDecoder.timed_events = True, True
    sysm.loop.run()
    kv.close()
    sysm.close()
    return out


if __name__ == "__main__":
    print(json.dumps({"context_128k": case(1, 131072), "config1_4x4k": case(4, 4096),
                      "context_128k_cap148": case(1, 131072, cap=148)}, indent=1))
