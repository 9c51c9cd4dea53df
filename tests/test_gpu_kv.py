"""KV offload path on a real GPU: append -> evict to a
harvested peer slab (donor = the same GPU here) or host -> reload / per-layer
gather (K1), with revocation fallback.  Bytes are checked against the oracle's
content for every (layer, sequence, block) page."""
import numpy as np
import pytest
import torch

from oracle import harvest_oracle as O
from tests import refcheck

pytestmark = pytest.mark.gpu


def _mk(local_blocks=8, host_blocks=64, slab_blocks=4, donor_slabs=2, durability="LOSSY", order="LRU"):
    from paper_2602_00328_b200.kv import EvictionOrder, KVCacheManager, KVModelSpec, OffloadPolicy
    from paper_2602_00328_b200.runtime import Durability
    from paper_2602_00328_b200.system import HarvestSystem
    m = KVModelSpec("tiny", num_layers=4, kv_heads=2, head_dim=64)
    slab = slab_blocks * m.block_bytes
    sysm = HarvestSystem(0, donors=[0] if donor_slabs else [], donor_bytes=donor_slabs * slab,
                         host_bytes=1 << 20, local_bytes=1 << 20)
    kv = KVCacheManager(sysm, m, local_blocks, host_blocks, OffloadPolicy(EvictionOrder[order]),
                        slab_blocks=slab_blocks, durability=Durability[durability])
    return sysm, kv, m


def _check_all(kv, m):
    """Gather every layer of every block and compare with the oracle."""
    ids = sorted(kv.table)
    dst = torch.empty(len(ids) * m.page_bytes, dtype=torch.uint8, device="cuda")
    for layer in range(m.num_layers):
        kv.gather_layer(layer, ids, dst)
        kv.sys.engine.synchronize()
        got = dst.cpu().numpy().reshape(len(ids), m.page_bytes)
        for i, bid in enumerate(ids):
            b = kv.table[bid]
            want = O.content(O.kv_seed(layer, b.sequence_id, b.index), m.page_bytes)
            assert np.array_equal(got[i], want), (bid, layer, b.tier)


def test_append_evict_reload_roundtrip():
    from paper_2602_00328_b200.kv import KVTier
    sysm, kv, m = _mk()
    assert kv.append_kv(0, 16) == [0]                      # 16 tokens -> one block
    assert kv.append_kv(1, 17) == [1, 2]                   # 17 -> two blocks, second holds 1
    assert kv.table[2].entries == 1
    kv.append_kv(2, 16 * 10)                               # exceeds 8 local slots -> evictions
    tiers = [b.tier for b in kv.table.values()]
    assert tiers.count(KVTier.PEER_HBM) > 0
    assert sum(1 for t in tiers if t == KVTier.LOCAL_HBM) <= 8
    assert kv.sys.loop.log.of_kind("kv_evict")
    _check_all(kv, m)                                      # reads from local + peer
    plan = kv.reload([b.block_id for b in kv.table.values() if b.tier == KVTier.PEER_HBM][:3])
    assert len(plan["peer"]) == 3
    kv.sys.engine.synchronize()
    sysm.loop.run()
    _check_all(kv, m)
    assert refcheck.verify_release_ordering(sysm.loop.log) == []
    kv.close()
    sysm.close()


def test_lossy_revocation_recomputes_and_backed_falls_back_to_host():
    from paper_2602_00328_b200.kv import KVTier
    from paper_2602_00328_b200.runtime import RevokeReason
    for dur, want_tier in (("LOSSY", KVTier.NOT_MATERIALIZED), ("BACKED", KVTier.HOST_DRAM)):
        sysm, kv, m = _mk(durability=dur)
        kv.append_kv(0, 16 * 12)
        peer = [b for b in kv.table.values() if b.tier == KVTier.PEER_HBM]
        assert peer
        slab = kv.slabs[peer[0].slab]
        sysm.runtime.revoke(slab.handle, RevokeReason.EXTERNAL_RECLAIM)
        sysm.loop.run()
        assert all(kv.table[b.block_id].tier == want_tier for b in peer if b.slab == -1)
        plan = kv.reload([b.block_id for b in peer])
        if dur == "LOSSY":
            assert plan["recompute"]
        else:
            assert plan["host"] and not plan["recompute"]
        kv.sys.engine.synchronize()
        sysm.loop.run()
        _check_all(kv, m)                                  # correctness independent of the peer tier
        assert refcheck.verify_release_ordering(sysm.loop.log) == []
        kv.close()
        sysm.close()


def test_no_peer_capacity_goes_to_host():
    from paper_2602_00328_b200.kv import KVTier
    sysm, kv, m = _mk(donor_slabs=0)
    kv.append_kv(0, 16 * 12)
    assert not any(b.tier == KVTier.PEER_HBM for b in kv.table.values())
    assert kv.stats["evict_host"] >= 4 and kv.stats["evict_peer"] == 0
    _check_all(kv, m)
    kv.close()
    sysm.close()


@pytest.mark.parametrize("chunk", [1, 3, 5])
def test_chunked_launches_evict_and_reload(chunk):
    """evict()/reload() launch K1 every `launch_chunk_blocks` blocks, pipelined
    with the host-side resolution; bytes, tiers and the drain bookkeeping must
    not depend on the chunking (peer and host sources mixed within a call)."""
    from paper_2602_00328_b200.kv import KVTier
    sysm, kv, m = _mk(local_blocks=16, slab_blocks=2, donor_slabs=2, durability="BACKED")
    kv.launch_chunk_blocks = chunk
    kv.timing = []
    kv.append_kv(0, 16 * 16)
    moves = kv.evict(12 * m.block_bytes)                   # 4 blocks to peer (+host copies), 8 to host
    assert len(moves) == 12
    assert {t for _, _, t in moves} == {"PeerHBM", "HostDRAM"}
    n_launch = len(kv.timing)
    assert n_launch >= 2 if chunk < 12 else n_launch == 1
    _check_all(kv, m)
    ids = [b.block_id for b in kv.table.values() if b.tier != KVTier.LOCAL_HBM]
    kv.timing = []
    plan = kv.reload(ids)
    assert plan["peer"] and plan["host"] and not plan["recompute"]
    assert len(kv.timing) == -(-len(ids) // chunk)
    kv.sys.engine.synchronize()
    sysm.loop.run()
    assert all(kv.table[i].tier == KVTier.LOCAL_HBM for i in ids)
    _check_all(kv, m)
    assert refcheck.verify_release_ordering(sysm.loop.log) == []
    kv.close()
    sysm.close()


@pytest.mark.parametrize("seed", range(50))
def test_kv_correctness_independence(seed):
    """SPEC.md acceptance #3, KV half: random append / evict / reload with every
    peer slab revoked at a random point (Lossy and Backed sequences mixed);
    the final bytes of every page equal the zero-peer-capacity result, i.e.
    the oracle content of (layer, sequence, block)."""
    import random
    from paper_2602_00328_b200.kv import KVTier
    from paper_2602_00328_b200.runtime import Durability, RevokeReason
    rng = random.Random(seed)
    sysm, kv, m = _mk(local_blocks=12, host_blocks=256, slab_blocks=2, donor_slabs=3,
                      durability=rng.choice(["LOSSY", "BACKED"]))
    kv.launch_chunk_blocks = rng.choice([1, 2, 64])
    revoked = 0
    for _ in range(12):
        r = rng.random()
        if r < 0.4:
            kv.append_kv(rng.randrange(4), rng.randint(1, 40), durability=rng.choice(list(Durability)))
        elif r < 0.6 and kv.table:
            kv.evict(rng.randint(1, 4) * m.block_bytes)
        elif r < 0.8 and kv.table:
            ids = rng.sample(sorted(kv.table), min(len(kv.table), rng.randint(1, 6)))
            kv.reload(ids)
        live = [s for s in kv.slabs if s.live]
        if live and rng.random() < 0.5:
            sysm.runtime.revoke(rng.choice(live).handle, RevokeReason.EXTERNAL_RECLAIM)
            revoked += 1
        sysm.loop.poll()
    for s in kv.slabs:  # every remaining slab is revoked too
        if s.live:
            sysm.runtime.revoke(s.handle, RevokeReason.EXTERNAL_RECLAIM)
            revoked += 1
    kv.sys.engine.synchronize()
    sysm.loop.run()
    assert all(b.tier != KVTier.PEER_HBM for b in kv.table.values())
    lost = sorted(i for i, b in kv.table.items() if b.tier == KVTier.NOT_MATERIALIZED)
    for k in range(0, len(lost), 6):   # Lossy-lost blocks are recomputed (local room for 6 at a time)
        kv.reload(lost[k:k + 6])
    kv.sys.engine.synchronize()
    sysm.loop.run()
    _check_all(kv, m)
    assert refcheck.verify_release_ordering(sysm.loop.log) == []
    kv.close()
    sysm.close()


def test_gather_layer_reads_are_drained_before_release():
    """gather_layer's peer reads join the slab's drain set: a revocation issued
    right after the launch finishes only after the gather, whose bytes are
    intact (the VMM chunks are unmapped only after the drain)."""
    import numpy as np
    from paper_2602_00328_b200.kv import KVTier
    from paper_2602_00328_b200.runtime import RevokeReason
    sysm, kv, m = _mk(local_blocks=4, slab_blocks=4, donor_slabs=2, durability="BACKED")
    kv.append_kv(0, 16 * 8)
    peer = [b.block_id for b in kv.table.values() if b.tier == KVTier.PEER_HBM]
    assert peer
    dst = torch.empty(len(peer) * m.page_bytes, dtype=torch.uint8, device="cuda")
    for layer in range(m.num_layers):
        kv.gather_layer(layer, peer, dst)
        for s in kv.slabs:
            if s.live:
                sysm.runtime.revoke(s.handle, RevokeReason.EXTERNAL_RECLAIM)
        sysm.loop.run()                       # waits for the gather, then releases
        got = dst.cpu().numpy().reshape(len(peer), m.page_bytes)
        for i, bid in enumerate(peer):
            b = kv.table[bid]
            want = O.content(O.kv_seed(layer, b.sequence_id, b.index), m.page_bytes)
            assert np.array_equal(got[i], want), (layer, bid)
        if layer == 0:                        # later layers read the Backed host copies
            assert all(kv.table[bid].tier == KVTier.HOST_DRAM for bid in peer)
    assert refcheck.verify_release_ordering(sysm.loop.log) == []
    kv.close()
    sysm.close()


def test_slab_emptied_while_revoking_is_left_to_the_revocation():
    """A slab whose revoke is still draining (a read holds it) can be emptied
    by a reload: the manager must neither free it (it is not LIVE) nor place
    new blocks in it; the revocation finishes it once the read ends."""
    from paper_2602_00328_b200.kv import KVTier
    from paper_2602_00328_b200.runtime import RevokeReason
    sysm, kv, m = _mk(local_blocks=8, slab_blocks=2, donor_slabs=2, durability="BACKED")
    kv.append_kv(0, 16 * 10)                              # 2 blocks evicted into a slab
    peer = [b for b in kv.table.values() if b.tier == KVTier.PEER_HBM]
    assert peer
    slab = kv.slabs[peer[0].slab]
    hold = sysm.runtime.begin_reads([slab.handle])         # an in-flight read keeps the drain open
    sysm.runtime.revoke(slab.handle, RevokeReason.EXTERNAL_RECLAIM)
    assert sysm.runtime.is_draining(slab.handle)
    kv.reload([b.block_id for b in peer if b.slab == kv.slabs.index(slab)])   # empties it: no free, no raise
    kv.append_kv(1, 16 * 4)                                # evictions must avoid the draining slab
    assert all(b.slab != kv.slabs.index(slab) for b in kv.table.values() if b.tier == KVTier.PEER_HBM)
    sysm.runtime.end_reads(hold)
    sysm.loop.run()
    assert sysm.runtime.lookup(slab.handle) is None and not slab.live
    _check_all(kv, m)
    assert refcheck.verify_release_ordering(sysm.loop.log) == []
    kv.close()
    sysm.close()


def test_evict_running_out_of_host_slots_leaves_a_consistent_table():
    """TierExhausted partway through evict() must not leave table
    entries pointing at pages that were never written, nor leak the slab slot
    taken for the failing victim.  Here Backed blocks go to a peer slab and
    need a host copy each; the host tier holds only 3, so the 4th victim
    fails.  The first 3 are complete (bytes equal the oracle's), the failing
    one is still local, and no slot is double-booked."""
    from paper_2602_00328_b200.kv import KVTier, TierExhausted
    sysm, kv, m = _mk(local_blocks=8, host_blocks=3, slab_blocks=8, donor_slabs=1, durability="BACKED")
    kv.append_kv(0, 16 * 8)                        # fills local HBM, no eviction yet
    free_before = sum(len(s.free) for s in kv.slabs)
    with pytest.raises(TierExhausted):
        kv.evict(6 * m.block_bytes)
    peer = [b for b in kv.table.values() if b.tier == KVTier.PEER_HBM]
    local = [b for b in kv.table.values() if b.tier == KVTier.LOCAL_HBM]
    assert len(peer) == 3 and len(local) == 5
    assert all(b.host_slot is not None for b in peer)
    assert all(b.host_slot is None for b in local)
    # slab slots: exactly the 3 moved blocks are booked
    booked = sum(len(s.blocks) for s in kv.slabs)
    assert booked == 3 and sum(len(s.free) for s in kv.slabs) + booked == len(kv.slabs) * 8
    assert free_before == 0 or free_before - 3 == sum(len(s.free) for s in kv.slabs)
    # local slots: the local blocks' slots are not on the free list
    assert not ({b.slot for b in local} & set(kv.local_free))
    _check_all(kv, m)
    kv.close()
    sysm.close()


def test_host_copy_dropped_when_a_reloaded_block_grows():
    """after reload, append_kv adds entries to the tail block; its
    old host copy no longer matches and must not be served later.  The copy
    is dropped and the next evict writes a fresh one."""
    from paper_2602_00328_b200.kv import KVTier
    sysm, kv, m = _mk(local_blocks=8, host_blocks=16, slab_blocks=4, donor_slabs=0, durability="BACKED")
    kv.append_kv(0, 20)                            # blocks 0 (16) and 1 (4 entries, the open tail)
    kv.evict(8 * m.block_bytes)                    # both to host (no donors)
    tail = kv.table[1]
    assert tail.tier == KVTier.HOST_DRAM and tail.host_slot is not None
    old_slot = tail.host_slot
    kv.append_kv(0, 3)                             # reloads the tail, then grows it
    assert tail.tier == KVTier.LOCAL_HBM and tail.entries == 7
    assert tail.host_slot is None and old_slot in kv.host_free
    writes0 = kv.stats["evict_host"]
    kv.evict(8 * m.block_bytes)
    assert tail.tier == KVTier.HOST_DRAM and tail.host_slot is not None
    assert kv.stats["evict_host"] > writes0
    _check_all(kv, m)
    kv.close()
    sysm.close()


def test_fallback_on_measured_costs():
    """§8(f)4: measure the host link (calibrate() refit of real fetch
    latencies) and a recompute curve (chunked prefill of a small dense
    shape) on this GPU, hand them to the KV manager, and check its decision
    equals the SPEC rule evaluated on the same measured numbers on both sides
    of the solved crossover."""
    from paper_2602_00328_b200.costs import DenseShape, fallback_crossover, fetch_wins, measure_host_link, \
        measure_recompute
    from paper_2602_00328_b200.kv import KVBlock, KVTier
    from paper_2602_00328_b200.runtime import Durability
    sysm, kv, m = _mk(durability="BACKED")
    from paper_2602_00328_b200.pool import HostTier
    ht = HostTier(16 << 20)
    link, fit = measure_host_link(ht, 0)
    assert 1e-6 < link.fixed_cost < 1e-3 and 10e9 < link.bandwidth < 80e9, fit
    shape = DenseShape("tiny", num_layers=2, hidden=512, q_heads=8, kv_heads=2, head_dim=64, intermediate=1024)
    curve = measure_recompute(shape, chunks=(16, 64, 256), iters=2)
    assert all(t > 0 for _, t in curve.points)
    kv.set_costs(host_link=link, recompute=curve)
    out = fallback_crossover(link, m.bytes_per_entry, curve, max_entries=4096)
    probe = [1, 16, 64, 256, 4096]
    for f in out["flips"]:
        probe += list(f.values())
    for e in probe:
        b = KVBlock(0, 0, 0, e, Durability.BACKED, KVTier.NOT_MATERIALIZED, host_slot=0)
        want = "FetchFromHost" if fetch_wins(link, e, m.bytes_per_entry, curve) else "Recompute"
        assert kv.resolve_fallback(b) == want
    ht.close()
    kv.close()
    sysm.close()


def test_evict_reload_as_coalesced_runs_bit_exact():
    """Blocks evicted together hold consecutive host slots, so evict and
    reload go out as per-layer runs (F.layer_runs) through the engine per
    source -- the copy engine to and from the pinned host tier once a run
    reaches 1 MiB.  64 KiB pages (Llama-3-8B geometry, 2 layers), 48 blocks:
    3 MiB runs.  Every page equals the oracle's before, after the evict (read
    from the host copy) and after the reload."""
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.kv import KVCacheManager, KVModelSpec, KVTier
    from paper_2602_00328_b200.runtime import Durability
    from paper_2602_00328_b200.system import HarvestSystem
    m = KVModelSpec("runs", num_layers=2, kv_heads=8, head_dim=128)
    assert m.page_bytes == 65536
    sysm = HarvestSystem(0, host_bytes=1, local_bytes=1)
    kv = KVCacheManager(sysm, m, local_blocks=64, host_blocks=64, slab_blocks=8, durability=Durability.BACKED)
    kv.append_kv(0, 16 * 48)
    ids = list(kv.seq_blocks[0])
    bases, strides, _h = kv.page_table(ids)
    n = len(ids)
    runs = F.layer_runs(bases, strides, np.arange(n, dtype=np.uint64) * np.uint64(m.page_bytes),
                        np.zeros(n, dtype=np.uint64), m.page_bytes, m.num_layers)
    assert runs is not None and len(runs[0]) == m.num_layers   # one run per layer in the cache
    _check_all(kv, m)
    kv.evict(48 * m.block_bytes)
    assert all(kv.table[b].tier == KVTier.HOST_DRAM for b in ids)
    slots = [kv.table[b].host_slot for b in ids]
    assert slots == sorted(slots) and slots[-1] - slots[0] == 47   # consecutive host slots
    _check_all(kv, m)
    kv.reload(ids)
    kv.sys.engine.synchronize()
    assert all(kv.table[b].tier == KVTier.LOCAL_HBM for b in ids)
    local = [kv.table[b].slot for b in ids]
    assert local == sorted(local)                            # ascending slots: coalescible
    _check_all(kv, m)
    kv.close()
    sysm.close()
