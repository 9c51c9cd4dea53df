"""The reference's acceptance criteria that apply to the runtime,
run against the B200 package on its modeled engine (CPU, no GPU):

 #1  allocator oracle: 1,000 random free-list/request instances, best fit ==
     exhaustive minimal-leftover search;
 #2  revocation ordering: >= 10,000-event random schedules with concurrent
     transfers and revocations, zero drain-before-free / invalidate-before-notify
     violations (verify.py:25-69) and no runtime-initiated transfers;
 #3  correctness independence (MoE, Backed): adversarial runs that revoke every
     peer allocation at a random time after it is made (the reference's
     on_alloc adversary) deliver exactly the content of a
     zero-peer-capacity run, for 50 seeds (the KV half is GPU-tier:
     tests/test_gpu_kv.py::test_kv_correctness_independence);
 #9  determinism: the same seed gives an identical event log;
 #10 resolve_fallback picks the cheaper modeled option on 100 cells.
"""
import random
import types

import pytest

from paper_2602_00328_b200 import memalloc as M
from paper_2602_00328_b200 import runtime as R
from paper_2602_00328_b200.events import VirtualLoop
from paper_2602_00328_b200.interconnect import LinkKind, LinkSpec, transfer_time
from paper_2602_00328_b200.memalloc import Segment, Tier
from tests.refcheck import verify_no_runtime_writeback, verify_release_ordering
from tests.test_runtime_parity import topo

MiB = 1 << 20


# ---------------------------------------------------------------- #1
def _exhaustive(free_list, size):
    fits = [(s.size - size, s.base) for s in free_list if s.size >= size]
    return min(fits)[1] if fits else None


def test_allocator_oracle_1000_instances():
    rng = random.Random(1)
    for _ in range(1000):
        usable = rng.choice([4096, 1 << 20, 1 << 34])
        st = M.init_device(M.DeviceSpec(1, Tier.PEER_HBM, usable))
        live = []
        for _ in range(rng.randint(0, 25)):  # a random free list
            if live and rng.random() < 0.45:
                M.free_segment(st, live.pop(rng.randrange(len(live))))
            else:
                seg = M.alloc_best_fit(st, rng.randint(1, max(1, usable // rng.choice([3, 10, 50]))))
                if seg is not None:
                    live.append(seg)
        size = rng.randint(1, max(1, usable // rng.choice([2, 8, 64])))
        want = _exhaustive(st.free_list, size)
        got = M.alloc_best_fit(st, size)
        assert (None if got is None else got.base) == want
        M.check_invariants(st)


# ---------------------------------------------------------------- #2
def test_revocation_ordering_10k_events():
    loop = VirtualLoop()
    rt = R.HarvestRuntime(loop, topo([(256 * MiB, 0, 0), (192 * MiB, 8 * MiB, 8 * MiB), (128 * MiB, 0, 0)]))
    hid = 4
    rng = random.Random(2)
    handles = []

    def act():
        r = rng.random()
        live = [h for h in handles if h.key() in rt.placement and rt.placement[h.key()].state == R._State.LIVE]
        if r < 0.3 or not live:
            h = rt.harvest_alloc(rng.randint(1, 24 * MiB),
                                 R.AllocationHints(durability=rng.choice(list(R.Durability))))
            if h is not None:
                handles.append(h)
                rt.harvest_register_cb(h, lambda hh, reason: None)
                rt.app_transfer(src=(hid, Segment(0, h.size)), dst=(h.device_id, Segment(h.base, h.size)),
                                size=h.size, tag=("obj", h.key()), handle=h, payload=rng.getrandbits(64))
        elif r < 0.65:
            h = rng.choice(live)
            if rt.lookup(h) is not None and rt.has_content(h):
                for _ in range(rng.randint(1, 3)):  # concurrent reads that must drain
                    rt.app_transfer(src=(h.device_id, Segment(h.base, h.size)), dst=(0, Segment(0, h.size)),
                                    size=h.size, tag=None, handle=h)
        elif r < 0.8:
            rt.revoke(rng.choice(live), rng.choice(list(R.RevokeReason)))
        elif r < 0.9:
            rt.harvest_free(rng.choice(live))
        else:
            dev = rng.choice([1, 2, 3])
            if rng.random() < 0.5:
                rt.external_reclaim(dev, rng.randint(0, 64 * MiB), order=rng.choice(["lru", "fifo"]))
            else:
                rt.set_availability(dev, rng.randint(0, 256 * MiB))

    t = 0.0
    for _ in range(5000):
        t += rng.expovariate(1 / 2e-4)
        loop.schedule_at(t, act)
    loop.run()
    log = loop.log
    assert len(log) >= 10_000
    assert log.of_kind("revoke_begin") and log.of_kind("transfer_complete")
    assert verify_release_ordering(log) == []
    assert verify_no_runtime_writeback(log) == []


# ---------------------------------------------------------------- #3 and #9
def _moe_run(seed, peer_capacity, adversarial):
    """Modeled decode through the product's placement (rebalance) and fetch plan
    (ExpertFetcher.plan); every fetch issued with app_transfer like
    _issue_fetches (moe.py:298-313).  Returns (deliveries, log)."""
    from paper_2602_00328_b200.moe import (ExpertFetcher, ExpertResidency, ExpertStore, MoEProfile, expert_content,
                                           rebalance, topk_routing)
    import numpy as np
    m = MoEProfile("accept", num_layers=3, num_experts=8, top_k=2, expert_size=1 * MiB)
    loop = VirtualLoop()
    cap = max(1, peer_capacity)
    rt = R.HarvestRuntime(loop, topo([(cap, 0, 0), (cap, 0, 0)]))
    hid = 3
    if not peer_capacity:
        for d in (1, 2):
            rt.set_availability(d, 0)
    rng = random.Random(seed)
    if adversarial:  # revoke every allocation at a random time after it is made
        rt.on_alloc = lambda h: loop.schedule(rng.uniform(0, 5e-3), rt.revoke, h, R.RevokeReason.POLICY)
    res = ExpertResidency(m)
    store = ExpertStore(m, hid)
    fetcher = ExpertFetcher(rt, m, res, store)
    counts = np.ones((m.num_layers, m.num_experts), dtype=np.int64)
    routes = topk_routing(m, tokens=4, steps=8, seed=seed)
    deliveries, errors = {}, []

    def stage(s, layer):
        for e, tier in fetcher.plan(layer, routes[s][layer]):
            want = expert_content(m, layer, e)
            if tier == "peer":
                h = fetcher.handles[(layer, e)]
                src, kw = (h.device_id, Segment(h.base, h.size)), dict(handle=h)
            else:
                src, kw = (hid, store.host_segment(layer, e)), dict(payload=want)

            def done(_x, content, key=(s, layer, e), want=want):
                deliveries[key] = content
                if content != want:
                    errors.append(key)
            rt.app_transfer(src=src, dst=(0, Segment(0, m.expert_size)), size=m.expert_size,
                            tag=("expert", layer, e), on_complete=done, **kw)

    def step(s):
        rebalance(loop, rt, m, res, counts, hid, store=store)  # re-place whatever was revoked
        for layer in range(m.num_layers):
            loop.schedule(layer * 1e-3, stage, s, layer)

    for s in range(len(routes)):
        loop.schedule_at(s * 4e-3, step, s)
    loop.run()
    assert errors == []
    return deliveries, loop.log


@pytest.mark.parametrize("seed", range(50))
def test_moe_correctness_independence_50_seeds(seed):
    base, _ = _moe_run(seed, 0, adversarial=False)
    got, log = _moe_run(seed, 12 * MiB, adversarial=True)
    assert got == base
    assert log.of_kind("revoke_begin")                    # the adversary did act
    assert any(r.data.get("handle") for r in log.of_kind("transfer_start"))  # and peers were read
    assert verify_release_ordering(log) == []
    assert verify_no_runtime_writeback(log) == []


def test_determinism_same_seed_same_log():
    a, la = _moe_run(11, 12 * MiB, adversarial=True)
    b, lb = _moe_run(11, 12 * MiB, adversarial=True)
    assert a == b
    assert [repr(r) for r in la] == [repr(r) for r in lb]


# ---------------------------------------------------------------- #10
def test_resolve_fallback_picks_the_cheaper_option_100_cells():
    from paper_2602_00328_b200.kv import KVBlock, KVCacheManager, KVModelSpec
    link = LinkSpec(LinkKind.HOST_LINK, 10e-6, 55e9, endpoints=(0, 9))
    rng = random.Random(10)
    models = [KVModelSpec("llama-3-8b", 32, 8, 128), KVModelSpec("mistral", 88, 8, 128),
              KVModelSpec("kimi", 61, 1, 576), KVModelSpec("tiny", 2, 1, 64)]
    cells = 0
    for m0 in models:
        for _ in range(25):
            rate = 10 ** rng.uniform(-9, -4)
            m = KVModelSpec(m0.name, m0.num_layers, m0.kv_heads, m0.head_dim, recompute_time_per_entry=rate)
            entries = rng.randint(1, 16)
            stub = types.SimpleNamespace(m=m)
            blk = KVBlock(0, 0, 0, entries, R.Durability.BACKED, host_slot=0)
            got = KVCacheManager.resolve_fallback(stub, blk, host_link=link)
            fetch, recompute = transfer_time(link, entries * m.bytes_per_entry), entries * rate
            assert got == ("FetchFromHost" if fetch <= recompute else "Recompute")
            # a block without a host copy can only be recomputed
            lossy = KVBlock(1, 0, 0, entries, R.Durability.LOSSY, host_slot=None)
            assert KVCacheManager.resolve_fallback(stub, lossy, host_link=link) == "Recompute"
            cells += 1
    assert cells == 100


def test_kv_residency_version_tracks_every_placement_change():
    """kv.residency_version (the page-table cache key of kv_decode) must move
    on every change of where a block's pages are, and only then."""
    from paper_2602_00328_b200 import kv as K
    b = K.KVBlock(0, 0, 0, 16, R.Durability.LOSSY)
    v = K.residency_version()
    b.last_access = 1.0
    b.entries = 8
    assert K.residency_version() == v
    for name, value in (("tier", K.KVTier.PEER_HBM), ("slot", 3), ("slab", 1), ("host_slot", 7)):
        setattr(b, name, value)
        assert K.residency_version() > v, name
        v = K.residency_version()
    s = K._Slab(None, 4096)
    assert K.residency_version() > v
    v = K.residency_version()
    s.blocks[0] = 0
    assert K.residency_version() == v
    s.live = False
    assert K.residency_version() > v
