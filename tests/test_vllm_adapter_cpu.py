"""The vLLM adapter binds to vLLM's own OffloadingHandler contract when vLLM is
installed (vllm/v1/kv_offload/worker/worker.py:26-75)."""
import inspect

import pytest


def test_adapter_implements_vllm_contract():
    from paper_2602_00328_b200 import vllm_adapter as v
    for name in ("transfer_async", "get_finished", "wait", "shutdown"):
        assert callable(getattr(v.HarvestPeerHandler, name))
    sig = inspect.signature(v.HarvestPeerHandler.transfer_async)
    assert list(sig.parameters) == ["self", "job_id", "spec"]
    if not v.HAVE_VLLM:
        pytest.skip("vLLM not installed")
    from vllm.v1.kv_offload.worker.worker import OffloadingHandler
    assert issubclass(v.HarvestPeerHandler, OffloadingHandler)
    assert v.PeerBlocks.medium() == "PEER" and v.GPUBlocks.medium() == "GPU"


class _Residency:
    """Stand-in for the worker's PeerBlockPool residency view."""

    def __init__(self):
        self.resident, self.released = set(), []

    def is_resident(self, b):
        return b in self.resident

    def release(self, b):
        self.resident.discard(b)
        self.released.append(b)


def _stored(mgr, res, keys):
    out = mgr.prepare_store(keys, None)
    ids = [int(x) for x in out.store_spec.block_ids]
    res.resident.update(ids)                      # what the handler's store job does
    mgr.complete_store(out.keys_to_store, None)
    return out, ids


def test_manager_store_lookup_load_lru_and_events():
    """OffloadingManager contract (vllm/v1/kv_offload/base.py:110-237)."""
    from paper_2602_00328_b200.vllm_adapter import HarvestOffloadingManager
    res = _Residency()
    mgr = HarvestOffloadingManager(3, residency=res, enable_events=True)
    out = mgr.prepare_store([b"a", b"b"], None)
    assert out.keys_to_store == [b"a", b"b"] and out.evicted_keys == []
    assert mgr.lookup(b"a", None) is None                       # store in flight: retry
    res.resident.update(int(x) for x in out.store_spec.block_ids)
    mgr.complete_store([b"a", b"b"], None)
    assert mgr.lookup(b"a", None) is True and mgr.lookup(b"zz", None) is False
    assert mgr.prepare_store([b"a"], None).keys_to_store == []  # already stored
    spec = mgr.prepare_load([b"a"], None)
    assert spec.medium() == "PEER" and len(spec.block_ids) == 1
    mgr.touch([b"a"], None)                                     # b is now the LRU entry
    _, ids_c = _stored(mgr, res, [b"c"])
    out = mgr.prepare_store([b"d"], None)                       # full: evicts b (a is being loaded)
    assert out.evicted_keys == [b"b"]
    mgr.complete_store([b"d"], None, success=False)             # failed store: d is dropped
    assert mgr.lookup(b"d", None) is False
    mgr.complete_load([b"a"], None)
    ev = list(mgr.take_events())
    assert [(e.keys, e.removed) for e in ev] == [([b"a", b"b"], False), ([b"c"], False), ([b"b"], True)]
    assert list(mgr.take_events()) == []


def test_manager_revocation_is_a_lookup_miss():
    """A peer block whose slab was revoked is a MISS (vLLM recomputes): the
    entry is dropped, its id recycled, a removed event emitted.  A block
    still being loaded is not dropped under the reader."""
    from paper_2602_00328_b200.vllm_adapter import HarvestOffloadingManager
    res = _Residency()
    mgr = HarvestOffloadingManager(2, residency=lambda: res, enable_events=True)
    _, ids = _stored(mgr, res, [b"x", b"y"])
    list(mgr.take_events())
    mgr.prepare_load([b"y"], None)
    res.resident.clear()                                        # the slab was revoked
    assert mgr.lookup(b"x", None) is False
    assert mgr.lookup(b"y", None) is False                      # miss, but kept until its load completes
    assert mgr.stats["revoked_misses"] == 1
    assert [(e.keys, e.removed) for e in mgr.take_events()] == [([b"x"], True)]
    out, ids2 = _stored(mgr, res, [b"x"])                        # stored again in the recycled id
    assert ids2 == [ids[0]] and mgr.lookup(b"x", None) is True


def test_spec_registered_and_built_by_the_factory():
    """OffloadingSpecFactory.create_spec resolves "HarvestOffloadingSpec"
    (vllm/v1/kv_offload/factory.py:35-58) and sizes the peer block id space
    from peer_bytes_to_use and the KV cache's bytes per block."""
    v = pytest.importorskip("vllm")
    import torch
    from paper_2602_00328_b200 import vllm_adapter as A
    from vllm.config import DeviceConfig, KVTransferConfig, VllmConfig
    from vllm.v1.kv_cache_interface import FullAttentionSpec, KVCacheConfig, KVCacheGroupSpec, KVCacheTensor
    from vllm.v1.kv_offload.factory import OffloadingSpecFactory
    assert A.register_with_vllm() and "HarvestOffloadingSpec" in OffloadingSpecFactory._registry
    spec = FullAttentionSpec(16, num_kv_heads=8, head_size=128, dtype=torch.float16)
    L, nb = 4, 64
    kcc = KVCacheConfig(num_blocks=nb, kv_cache_tensors=[KVCacheTensor(size=spec.page_size_bytes * nb,
                                                                       shared_by=[f"l{i}"]) for i in range(L)],
                        kv_cache_groups=[KVCacheGroupSpec([f"l{i}" for i in range(L)], spec)])
    vc = VllmConfig(device_config=DeviceConfig(device="cpu"),
                    kv_transfer_config=KVTransferConfig(kv_connector="OffloadingConnector", kv_role="kv_both",
                                                        kv_connector_extra_config={
                                                            "spec_name": "HarvestOffloadingSpec",
                                                            "peer_bytes_to_use": 100 * L * spec.page_size_bytes}))
    s = OffloadingSpecFactory.create_spec(vc, kcc)
    assert isinstance(s, A.HarvestOffloadingSpec)
    assert s.block_bytes == L * spec.page_size_bytes and s.num_blocks == 100
    m = s.get_manager()
    assert isinstance(m, A.HarvestOffloadingManager) and m.num_blocks == 100
    assert m.lookup(b"k", None) is False
