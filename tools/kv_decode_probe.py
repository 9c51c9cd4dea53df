"""KV decode attention in one process with the KV in a self-donor VMM pool
(the "peer" tier on the same GPU: HBM, not NVLink) -- clean per-mode numbers
without the time sharing of the multi-rank stand-in.  Config 1 (4 x 4k) and
the 128k context, Llama-3-8B shapes.  Prints JSON: tokens/s and KV GB/s per
mode (gather / in place, eager / CUDA graph)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager  # noqa: E402
from paper_2602_00328_b200.kv_decode import KVAttentionDecoder  # noqa: E402
from paper_2602_00328_b200.runtime import Durability  # noqa: E402
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402


def timed(dec, steps=5):
    o = dec.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        o = dec.step()
    e1.record()
    e1.synchronize()
    return o, e0.elapsed_time(e1) / steps


def case(batch, ctx):
    m = LLAMA3_8B
    nblk = batch * ctx // m.block_tokens
    sysm = HarvestSystem(0, donors=[0], donor_bytes=(nblk // 64 + 2) * 64 * m.block_bytes, host_bytes=1,
                         local_bytes=1)
    kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=1, slab_blocks=64, durability=Durability.LOSSY,
                        content="fp16")
    for s in range(batch):
        kv.append_kv(s, ctx)
    nbytes = nblk * m.block_bytes
    out = {}
    seqs = list(range(batch))
    ref, ms = timed(KVAttentionDecoder(kv, seqs, q_heads=32, seed=1))
    out["local_gather"] = ms
    kv.evict(nbytes)
    for name, fused, graph in (("peer_gather", False, False), ("peer_gather_graph", False, True),
                               ("peer_in_place", True, False), ("peer_in_place_graph", True, True)):
        dec = KVAttentionDecoder(kv, seqs, q_heads=32, seed=1, fused=fused)
        if graph:
            dec.capture_graph()
        o, ms = timed(dec)
        assert torch.equal(o, ref), name
        out[name] = ms
        del dec
    sysm.loop.run()
    kv.close()
    sysm.close()
    return {k: {"ms_per_step": v, "tokens_per_s": batch / (v * 1e-3), "kv_GBps": nbytes / (v * 1e-3) / 1e9}
            for k, v in out.items()}


if __name__ == "__main__":
    if "--no-overlap" in sys.argv:   # A/B of the programmatic dependent launch of K5 across layers
        KVAttentionDecoder.overlap_layers = False
    if "--gather-pdl" in sys.argv:   # the same launch in gather mode
        KVAttentionDecoder.overlap_gather = True
    if "--grid" in sys.argv:         # A/B of the balanced (stream-K) K5 against the (split, head, seq) grid
        KVAttentionDecoder.balanced = False
    print(json.dumps({"overlap_layers": KVAttentionDecoder.overlap_layers, "balanced": KVAttentionDecoder.balanced,
                      "config1_4x4k": case(4, 4096), "context_128k": case(1, 131072),
                      "note": "self-donor VMM pool: the peer tier is this GPU's HBM; outputs of every mode "
                              "bit-identical to the all-local run"}, indent=1))
