"""vLLM OffloadingHandler contract (worker.py:26-75) over the harvested peer
tier: store GPU blocks to PEER, load them back to other GPU blocks, bytes
identical; a revoked slab makes the load complete with success=False."""
import pytest
import torch

from oracle import harvest_oracle as O

pytestmark = pytest.mark.gpu


def test_store_load_roundtrip_and_revocation():
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.runtime import RevokeReason
    from paper_2602_00328_b200.system import HarvestSystem
    from paper_2602_00328_b200.vllm_adapter import GPUBlocks, HarvestPeerHandler, PeerBlockPool, PeerBlocks
    L, nb, page, slab_blocks = 4, 32, 4096, 16
    sysm = HarvestSystem(0, donors=[0], donor_bytes=4 * slab_blocks * L * page, host_bytes=1, local_bytes=1)
    cache = torch.empty((L, nb, page), dtype=torch.uint8, device="cuda")
    seeds = [O.kv_seed(l, 0, b) for l in range(L) for b in range(nb)]
    F.fill_content(F.ptrs_tensor([cache[l, b].data_ptr() for l in range(L) for b in range(nb)], "cuda"),
                   F.ptrs_tensor([page] * (L * nb), "cuda"), seeds)
    torch.cuda.synchronize()
    ref = cache.clone()
    pool = PeerBlockPool(sysm.runtime, L, page, slab_blocks=slab_blocks)
    h = HarvestPeerHandler(sysm, cache, pool)
    gpu_src, peer_ids = list(range(10)), list(range(20, 30))       # spans slabs 1 and 2
    assert h.transfer_async(1, (GPUBlocks(gpu_src), PeerBlocks(peer_ids)))
    h.wait({1})
    res = h.get_finished()
    assert [r.job_id for r in res] == [1] and res[0].success and res[0].transfer_size == 10 * L * page
    cache[:, 10:20].zero_()
    assert h.transfer_async(2, (PeerBlocks(peer_ids), GPUBlocks(list(range(10, 20)))))
    h.wait({2})
    assert all(r.success for r in h.get_finished())
    torch.cuda.synchronize()
    assert torch.equal(cache[:, 10:20], ref[:, 0:10])
    # revoke the slab holding blocks 20..31 -> a load of them fails (Lossy)
    sysm.runtime.revoke(pool.slabs[1], RevokeReason.EXTERNAL_RECLAIM)
    sysm.loop.run()
    assert h.transfer_async(3, (PeerBlocks([20, 21]), GPUBlocks([0, 1])))
    h.wait({3})
    r3 = h.get_finished()
    assert r3 and not r3[0].success
    h.shutdown()
    sysm.close()
