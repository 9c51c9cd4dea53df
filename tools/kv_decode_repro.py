"""Single-process config-1 KV decode (gather + in-place) over a self-donor
VMM pool: for compute-sanitizer runs of the K1 + K5 path at bench shapes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200.kv import LLAMA3_8B, KVCacheManager  # noqa: E402
from paper_2602_00328_b200.kv_decode import KVAttentionDecoder  # noqa: E402
from paper_2602_00328_b200.runtime import Durability  # noqa: E402
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402


def main():
    batch, ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 4, int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    m = LLAMA3_8B
    nblk = batch * ctx // m.block_tokens
    sysm = HarvestSystem(0, donors=[0], donor_bytes=(nblk // 64 + 2) * 64 * m.block_bytes, host_bytes=1,
                         local_bytes=1)
    kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=1, slab_blocks=64, durability=Durability.LOSSY,
                        content="fp16")
    for s in range(batch):
        kv.append_kv(s, ctx)
    dec = KVAttentionDecoder(kv, list(range(batch)), q_heads=32, seed=1)
    a = dec.step()
    kv.evict(nblk * m.block_bytes)
    b = dec.step()
    f = KVAttentionDecoder(kv, list(range(batch)), q_heads=32, seed=1, fused=True)
    for _ in range(3):
        c = f.step()
    torch.cuda.synchronize()
    print("equal", torch.equal(a, b), torch.equal(b, c), "finite", bool(torch.isfinite(c).all()))
    kv.close()
    sysm.close()


if __name__ == "__main__":
    main()
