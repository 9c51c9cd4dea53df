"""vLLM OffloadingHandler contract (worker.py:26-75) over the harvested peer
tier: store GPU blocks to PEER, load them back to other GPU blocks, bytes
identical; a revoked slab makes the load complete with success=False."""
import numpy as np
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


def _spec(L, nb, peer_blocks, tensor_sizes):
    import torch as T
    from vllm.config import DeviceConfig, KVTransferConfig, VllmConfig
    from vllm.v1.kv_cache_interface import FullAttentionSpec, KVCacheConfig, KVCacheGroupSpec, KVCacheTensor
    from vllm.v1.kv_offload.factory import OffloadingSpecFactory
    from paper_2602_00328_b200 import vllm_adapter as A
    A.register_with_vllm()
    spec = FullAttentionSpec(16, num_kv_heads=2, head_size=64, dtype=T.float16)
    kcc = KVCacheConfig(num_blocks=nb, kv_cache_tensors=[KVCacheTensor(size=s * nb, shared_by=[f"l{i}"])
                                                         for i, s in enumerate(tensor_sizes)],
                        kv_cache_groups=[KVCacheGroupSpec([f"l{i}" for i in range(L)], spec)])
    vc = VllmConfig(device_config=DeviceConfig(device="cuda"),
                    kv_transfer_config=KVTransferConfig(
                        kv_connector="OffloadingConnector", kv_role="kv_both",
                        kv_connector_extra_config={"spec_name": "HarvestOffloadingSpec", "slab_blocks": 8,
                                                   "peer_bytes_to_use": peer_blocks * sum(tensor_sizes)}))
    return OffloadingSpecFactory.create_spec(vc, kcc)


@pytest.mark.parametrize("layout", ["stacked", "split_kv"])
def test_spec_manager_and_handler_store_revoke_miss_load(layout):
    """§8(f)1 end to end through vLLM's own factory: HarvestOffloadingSpec ->
    manager (scheduler side) + handler (worker side) over CanonicalKVCaches.
    store -> lookup hit -> slab revoked -> lookup MISS (vLLM would recompute)
    -> store again -> load into other GPU blocks; bytes equal the oracle's.
    "stacked": one [L, nb, page] buffer (K1 over the block table);
    "split_kv": separately allocated K and V tensors per layer with unequal
    pages (per-page pointer launch)."""
    pytest.importorskip("vllm")
    from vllm.v1.kv_offload.base import CanonicalKVCacheRef, CanonicalKVCaches, CanonicalKVCacheTensor, \
        GPULoadStoreSpec
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.runtime import RevokeReason
    L, nb = 3, 24
    if layout == "stacked":
        page = 4096
        big = torch.empty((L, nb, page), dtype=torch.int8, device="cuda")
        tensors = [big[i] for i in range(L)]
    else:
        sizes = [4096, 2048] * L                                     # K and V pages differ
        tensors = [torch.empty((nb, s), dtype=torch.int8, device="cuda") for s in sizes]
    psz = [t.shape[1] for t in tensors]
    s = _spec(L, nb, peer_blocks=16, tensor_sizes=psz)
    kv = CanonicalKVCaches(tensors=[CanonicalKVCacheTensor(t, p) for t, p in zip(tensors, psz)],
                           group_data_refs=[[CanonicalKVCacheRef(i, p) for i, p in enumerate(psz)]])
    handlers = list(s.get_handlers(kv))
    assert [(a.medium(), b.medium()) for a, b, _ in handlers] == [("GPU", "PEER"), ("PEER", "GPU")]
    h = handlers[0][2]
    assert h.block_form == (layout == "stacked")
    mgr = s.get_manager()
    seeds = [[O.kv_seed(t, 0, b) for b in range(nb)] for t in range(len(tensors))]
    F.fill_content(F.ptrs_tensor([tensors[t][b].data_ptr() for t in range(len(tensors)) for b in range(nb)], "cuda"),
                   F.ptrs_tensor([psz[t] for t in range(len(tensors)) for b in range(nb)], "cuda"),
                   [seeds[t][b] for t in range(len(tensors)) for b in range(nb)])
    torch.cuda.synchronize()
    keys = [bytes([k]) * 8 for k in range(10)]

    def gspec(ids):
        return GPULoadStoreSpec(ids, group_sizes=[len(ids)], block_indices=[0])

    def store(job, gpu_ids, ks):
        out = mgr.prepare_store(ks, None)
        assert out is not None and out.keys_to_store == ks
        assert h.transfer_async(job, (gspec(gpu_ids), out.store_spec))
        h.wait({job})
        assert all(r.success for r in h.get_finished())
        mgr.complete_store(ks, None)

    store(1, list(range(10)), keys)                                 # GPU blocks 0..9 -> peer
    assert all(mgr.lookup(k, None) for k in keys)
    # revoke the slab holding the first 8 peer blocks: those keys become misses
    s.system.runtime.revoke(s._pool.slabs[0], RevokeReason.EXTERNAL_RECLAIM)
    s.system.loop.run()
    hits = [mgr.lookup(k, None) for k in keys]
    assert hits.count(False) == 8 and hits.count(True) == 2
    assert mgr.stats["revoked_misses"] == 8
    store(2, list(range(8)), keys[:8])                              # recompute + offload again
    assert all(mgr.lookup(k, None) for k in keys)
    # load all 10 into GPU blocks 12..21
    for t in tensors:
        t[12:22].zero_()
    ld = mgr.prepare_load(keys, None)
    assert h.transfer_async(3, (ld, gspec(list(range(12, 22)))))
    h.wait({3})
    assert all(r.success for r in h.get_finished())
    mgr.complete_load(keys, None)
    torch.cuda.synchronize()
    for t in range(len(tensors)):
        got = tensors[t][12:22].cpu().numpy().view(np.uint8)
        for i in range(10):
            assert np.array_equal(got[i], O.content(seeds[t][i], psz[t])), (t, i)
    h.shutdown()
    s.system.close()
