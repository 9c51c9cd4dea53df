"""The expert fetch hook and the full-size configs, against the CPU oracle.

* ``ExpertFetcher.issue_fetches`` (moe.py:282-313) at the Qwen1.5-MoE expert
  size with LOCAL / PEER / HOST residency in one stage: the serving tier of
  every expert equals the oracle's restatement of the reference's decision
  (``O.stage_fetch_plan``), the staged bytes equal ``O.content`` of the
  expert's tag, and the per-fetch content check counts read_errors exactly
  as moe.py:315-319 does (including an injected corruption);
* a handle released between ``plan()`` and the launch: freed (lookup misses
  at once -> host copy, the branch of moe.py:300-302) or revoked (REVOKING
  is still readable -> peer read, and the release waits for it);
* K1 at BASELINE configs[0]'s full shape (1,024 x 64 KiB pages, block table
  [4, 256] = randperm(slots, seed 1)) from the host tier and from a VMM pool;
* one 157,286,400-B Phi-3.5-MoE expert moved by K2 from the host tier and
  from a pool, digest-checked against the oracle.
"""
import numpy as np
import pytest
import torch

from oracle import harvest_oracle as O

pytestmark = pytest.mark.gpu


def _qwen(layers=2):
    from paper_2602_00328_b200.moe import QWEN15_MOE_A27B, MoEProfile
    m = QWEN15_MOE_A27B
    return MoEProfile(m.name, layers, m.num_experts, m.top_k, m.expert_size, hidden=m.hidden,
                      intermediate=m.intermediate)


@pytest.fixture(scope="module")
def qwen_system():
    """Two Qwen layers: host tier authoritative, 20 experts placed on a donor
    pool (rebalance, the hottest first), 10 of layer 0 LOCAL."""
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, rebalance
    from paper_2602_00328_b200.system import HarvestSystem
    m = _qwen()
    L, E, S = m.num_layers, m.num_experts, m.expert_size
    sysm = HarvestSystem(0, donors=[0], donor_bytes=24 * S, host_bytes=L * E * S, local_bytes=1)
    store = ExpertStore(m, sysm.host_id, sysm.host)
    store.fill_host(0)
    res = ExpertResidency(m)
    counts = np.zeros((L, E), dtype=np.int64)
    counts[0, 10:30] = 100 - np.arange(20)           # layer-0 experts 10..29 are the hottest
    rebalance(sysm.loop, sysm.runtime, m, res, counts, sysm.host_id, max_migrations=20, store=store)
    sysm.loop.run()
    local = torch.empty(10 * S, dtype=torch.uint8, device="cuda")
    local_addr = np.zeros((L, E), dtype=np.uint64)
    for e in range(10):                                # layer-0 experts 0..9 resident in local HBM
        res.set_tier(0, e, Tier.LOCAL_HBM)
        local_addr[0, e] = local.data_ptr() + e * S
    fetcher = ExpertFetcher(sysm.runtime, m, res, store, local_addr=local_addr)
    fetcher.enable_content_check(store.host_digests(0))
    yield sysm, store, res, fetcher, m
    sysm.close()


def _oracle_plan(fetcher, layer, active):
    from paper_2602_00328_b200.memalloc import Tier
    tiers, live = {}, {}
    for e in active:
        ent = fetcher.residency.get(layer, int(e))
        tiers[int(e)] = {Tier.LOCAL_HBM: "local", Tier.PEER_HBM: "peer", Tier.HOST_DRAM: "host"}[ent.tier]
        live[int(e)] = ent.handle is not None and fetcher.rt.is_live(ent.handle)
    return O.stage_fetch_plan(tuple(int(e) for e in active), tiers, live)


def _staged_bytes_ok(m, layer, experts, staging, S):
    got = staging.cpu().numpy()
    for i, e in enumerate(experts):
        want = O.content(O.expert_seed(m.name, layer, int(e)), S)
        if not np.array_equal(got[i * S:(i + 1) * S], want):
            return False
    return True


def test_issue_fetches_mixed_tiers_match_oracle(qwen_system):
    sysm, store, res, fetcher, m = qwen_system
    S = m.expert_size
    active = np.array([0, 3, 9, 10, 12, 17, 25, 29, 30, 41, 59])   # 3 LOCAL, 5 PEER, 3 HOST
    plan = fetcher.plan(0, active)
    assert plan == _oracle_plan(fetcher, 0, active)
    assert [t for _, t in plan].count("peer") == 5 and [t for _, t in plan].count("host") == 3
    staging = torch.empty(len(active) * S, dtype=torch.uint8, device="cuda")
    dst = np.array([staging.data_ptr() + i * S for i in range(len(active))], dtype=np.uint64)
    reads0, err0 = fetcher.reads, fetcher.read_errors()
    batch = fetcher.issue_fetches(0, active, dst)
    torch.cuda.synchronize()
    sysm.loop.run()
    assert list(batch.experts) == [e for e, _ in plan]          # LOCAL skipped, order kept
    assert fetcher.reads - reads0 == len(plan)
    assert fetcher.read_errors() == err0 == 0
    # each fetched expert lands in the dst slot of its position in `active`
    got = staging.cpu().numpy()
    for i, e in enumerate(active):
        if fetcher.tier[0, e] == 0:
            continue
        want = O.content(O.expert_seed(m.name, 0, int(e)), S)
        assert np.array_equal(got[i * S:(i + 1) * S], want), e


def test_issue_fetches_counts_read_errors(qwen_system):
    """A corrupted donor copy is caught by the per-fetch check and only it."""
    sysm, store, res, fetcher, m = qwen_system
    S = m.expert_size
    from paper_2602_00328_b200 import _native as N
    h = res.get(0, 12).handle
    addr = sysm.runtime.address(h)
    import ctypes as C
    b = (C.c_uint8 * 1)()
    N.call("hv_memcpy_d2h", C.addressof(b), addr + 1000, 1, 0)
    torch.cuda.synchronize()
    N.call("hv_memset_d8", addr + 1000, b[0] ^ 0xFF, 1, 0)        # flip one byte of expert 12's peer copy
    torch.cuda.synchronize()
    active = np.array([11, 12, 13, 45])
    staging = torch.empty(len(active) * S, dtype=torch.uint8, device="cuda")
    dst = np.array([staging.data_ptr() + i * S for i in range(len(active))], dtype=np.uint64)
    err0 = fetcher.read_errors()
    fetcher.issue_fetches(0, active, dst)
    assert fetcher.read_errors() - err0 == 1
    assert list(fetcher.last_read_error_flags()[:4]) == [0, 1, 0, 0]
    # restore the copy from the authoritative host bytes (K2 host -> peer)
    from paper_2602_00328_b200 import fetch as F
    F.swap_blocks_batch([store.host.device_address(store.host_offset(0, 12))], [addr], [S], engine="ldg")
    torch.cuda.synchronize()


def test_released_between_plan_and_launch(qwen_system):
    """harvest_free: FREEING misses lookups at once -> the stale PEER table
    entry is served from the host copy (moe.py:300-302 / the product's
    re-check).  revoke: REVOKING stays readable -> peer read; the release
    completes only after the read drains, then the callback moves residency
    to the host tier."""
    sysm, store, res, fetcher, m = qwen_system
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.runtime import RevokeReason
    rt, S = sysm.runtime, m.expert_size
    active = np.array([14, 15, 16])
    plan = fetcher.plan(0, active)
    assert [t for _, t in plan] == ["peer"] * 3
    h_free, h_rev = res.get(0, 14).handle, res.get(0, 15).handle
    rt.harvest_free(h_free)
    rt.revoke(h_rev, RevokeReason.PRESSURE)
    assert not rt.is_live(h_free) and rt.is_live(h_rev)
    want = _oracle_plan(fetcher, 0, active)
    assert want == [(14, "host"), (15, "peer"), (16, "peer")]
    staging = torch.empty(3 * S, dtype=torch.uint8, device="cuda")
    dst = np.array([staging.data_ptr() + i * S for i in range(3)], dtype=np.uint64)
    src_before = fetcher.src_addr[0, active].copy()
    err0 = fetcher.read_errors()
    fetcher.issue_fetches(0, active, dst)
    assert fetcher.tier[0, 14] == 2 and fetcher.src_addr[0, 14] == fetcher.host_addr[0, 14]
    assert fetcher.src_addr[0, 15] == src_before[1]                # still read from the donor
    assert res.get(0, 15).tier == Tier.PEER_HBM                    # release waits for the drain
    torch.cuda.synchronize()
    sysm.loop.run()
    assert res.get(0, 15).tier == Tier.HOST_DRAM and not rt.is_live(h_rev)
    assert fetcher.read_errors() == err0
    assert _staged_bytes_ok(m, 0, active, staging, S)


def test_engine_per_source_mixed_batch():
    """hv_swap_blocks_batch AUTO: host-tier objects >= 1 MiB go to the copy
    engine on a side stream, the rest (HBM, small host pages) to the kernel,
    joined back into the caller's stream; bytes equal the oracle's."""
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.pool import HostTier
    sizes = [3 << 20, 65536, 17_301_504, 1000, (1 << 20) + 8, 4096]
    host = HostTier(sum(sizes))
    hbm = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
    seeds = [O.stable_hash64("mix", i) for i in range(len(sizes))]
    for i, (o, s) in enumerate(zip(offs, sizes)):
        host.view()[int(o):int(o) + s] = O.content(seeds[i], s)
    F.fill_content(F.ptrs_tensor([hbm.data_ptr() + int(o) for o in offs], "cuda"), F.ptrs_tensor(sizes, "cuda"),
                   seeds)
    # objects alternate host / HBM sources
    src = [host.device_address(int(o)) if i % 2 == 0 else hbm.data_ptr() + int(o) for i, o in enumerate(offs)]
    for engine in ("auto", "ce", "ldg"):
        out = torch.zeros(sum(sizes), dtype=torch.uint8, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            F.swap_blocks_batch(src, [out.data_ptr() + int(o) for o in offs], sizes, engine=engine, stream=s)
            got = out.cpu()                                      # ordered after the join on s
        got = got.numpy()
        for i, (o, sz) in enumerate(zip(offs, sizes)):
            assert np.array_equal(got[int(o):int(o) + sz], O.content(seeds[i], sz)), (engine, i)
    host.close()


@pytest.mark.parametrize("tier", ["host", "pool"])
def test_k1_config1_full_shape(tier):
    """BASELINE configs[0]: 4 sequences x 4k tokens, fp16, 8 KV heads x 128,
    16-token blocks = 1,024 pages of 64 KiB for one layer; block table
    [4, 256] = randperm(1024 slots, seed 1); K1 gathers into a
    contiguous [1024, 2, 16, 8, 128] fp16 buffer, bit-exact with the
    oracle's memcpy gather, both through the pointer form and the
    device-resolved table form."""
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.pool import HostTier, PeerPool
    page, slots = 2 * 16 * 8 * 128 * 2, 1024
    assert page == 65536
    if tier == "host":
        src_mem = HostTier(slots * page)
        base = src_mem.device_address(0)
    else:
        src_mem = PeerPool(0, slots * page, readers=[0])
        src_mem.commit(0, slots * page)
        base = src_mem.va
    seeds = [O.kv_seed(0, s // 256, s % 256) for s in range(slots)]
    F.fill_content(F.ptrs_tensor([base + s * page for s in range(slots)], "cuda"),
                   F.ptrs_tensor([page] * slots, "cuda"), seeds)
    table = torch.randperm(slots, generator=torch.Generator().manual_seed(1)).reshape(4, 256).to(torch.int32)
    flat = table.reshape(-1).numpy()
    dst = torch.empty(slots, 2, 16, 8, 128, dtype=torch.float16, device="cuda")
    F.kv_gather(F.ptrs_tensor([base + int(s) * page for s in flat], "cuda"), page, dst=dst.view(torch.uint8))
    torch.cuda.synchronize()
    host_copy = np.concatenate([O.content(sd, page) for sd in seeds])
    want = np.empty(slots * page, dtype=np.uint8)
    O.gather([host_copy.ctypes.data + int(s) * page for s in flat],
             [want.ctypes.data + i * page for i in range(slots)], [page] * slots, threads=8)
    assert np.array_equal(dst.view(torch.uint8).cpu().numpy().reshape(-1), want)
    dst2 = torch.zeros_like(dst)
    F.kv_gather_table(F.ptrs_tensor([base], "cuda"), F.ptrs_tensor([int(s) for s in flat], "cuda"), page,
                      dst=dst2.view(torch.uint8))
    torch.cuda.synchronize()
    assert torch.equal(dst2.view(torch.uint8), dst.view(torch.uint8))    # bytes (fp16 NaN != NaN)
    if tier == "pool":
        src_mem.decommit(0, slots * page)
    src_mem.close()


@pytest.mark.parametrize("tier", ["host", "pool"])
def test_k2_phi35_expert_full_size(tier):
    """One Phi-3.5-MoE expert (157,286,400 B, BASELINE configs[2]) through
    K2 and through the library's engine per source; digest equals the
    oracle's digest of the expert's content."""
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.moe import PHI35_MOE
    from paper_2602_00328_b200.pool import HostTier, PeerPool
    S = PHI35_MOE.expert_size
    assert S == 157_286_400
    seed = O.expert_seed(PHI35_MOE.name, 7, 3)
    if tier == "host":
        src_mem = HostTier(S)
        src = src_mem.device_address(0)
    else:
        src_mem = PeerPool(0, S, readers=[0])
        src_mem.commit(0, S)
        src = src_mem.va
    F.fill_content(F.ptrs_tensor([src], "cuda"), F.ptrs_tensor([S], "cuda"), [seed])
    want = O.content_digest(seed, S)
    dst = torch.empty(S, dtype=torch.uint8, device="cuda")
    sz = F.ptrs_tensor([S], "cuda")
    for engine in ("ldg", "ldg16", "tma"):
        dst.zero_()
        F.batch_copy(F.ptrs_tensor([src], "cuda"), F.ptrs_tensor([dst.data_ptr()], "cuda"), sz, engine=engine)
        assert int(F.digest(F.ptrs_tensor([dst.data_ptr()], "cuda"), sz).cpu().numpy().view(np.uint64)[0]) == want
    dst.zero_()
    F.swap_blocks_batch([src], [dst.data_ptr()], [S], engine="auto")
    assert int(F.digest(F.ptrs_tensor([dst.data_ptr()], "cuda"), sz).cpu().numpy().view(np.uint64)[0]) == want
    if tier == "pool":
        src_mem.decommit(0, S)
    src_mem.close()


@pytest.mark.parametrize("engine", ["auto", "ldg", "ldg16", "ce"])
def test_fetch_and_check_in_one_pass(engine):
    """hv_swap_blocks_batch_checked: the SM kernel copies and digests in one
    pass (copy-engine objects are digested after their copy); bytes equal
    the oracle's, digests are compared with the oracle's content digest, and
    a corrupted source is flagged -- exactly one read error, at its index."""
    from paper_2602_00328_b200 import _native as N
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.pool import HostTier
    sizes = [3 << 20, 65536, 17_301_504, 4096 + 8, (1 << 20) + 16, 8192, 2 << 20]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
    host = HostTier(sum(sizes))
    hbm = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
    seeds = [O.stable_hash64("chk", i) for i in range(len(sizes))]
    for i, (o, sz) in enumerate(zip(offs, sizes)):
        host.view()[int(o):int(o) + sz] = O.content(seeds[i], sz)
    F.fill_content(F.ptrs_tensor([hbm.data_ptr() + int(o) for o in offs], "cuda"), F.ptrs_tensor(sizes, "cuda"), seeds)
    torch.cuda.synchronize()
    src = np.array([host.device_address(int(o)) if i % 2 == 0 else hbm.data_ptr() + int(o)
                    for i, o in enumerate(offs)], dtype=np.uint64)
    out = torch.zeros(sum(sizes), dtype=torch.uint8, device="cuda")
    dst = np.array([out.data_ptr() + int(o) for o in offs], dtype=np.uint64)
    sz = np.array(sizes, dtype=np.uint64)
    exp = np.array([O.content_digest(sd, n) for sd, n in zip(seeds, sizes)], dtype=np.uint64)
    scratch = torch.zeros(len(sizes), dtype=torch.int64, device="cuda")
    flags = torch.zeros(len(sizes), dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()

    def run():
        N.call("hv_swap_blocks_batch_checked", src.ctypes.data, dst.ctypes.data, sz.ctypes.data, exp.ctypes.data,
               len(sizes), N.ENGINES[engine], 0, scratch.data_ptr(), flags.data_ptr(), err.data_ptr(), s.cuda_stream)
        s.synchronize()

    run()
    got = out.cpu().numpy()
    for i, (o, n) in enumerate(zip(offs, sizes)):
        assert np.array_equal(got[int(o):int(o) + n], O.content(seeds[i], n)), i
    assert int(err.item()) == 0 and int(flags.sum().item()) == 0
    assert [int(x) for x in scratch.cpu().numpy().view(np.uint64)] == [int(x) for x in exp]
    hbm[int(offs[3]) + 5] ^= 0x40                     # corrupt object 3 (an HBM source) at the source
    host.view()[int(offs[2]) + 12345] ^= 0x01         # and object 2 (a host-tier source)
    torch.cuda.synchronize()
    run()
    assert int(err.item()) == 2
    assert list(flags.cpu().numpy()) == [0, 0, 1, 1, 0, 0, 0]
    host.close()


def test_checked_fetch_many_ragged_objects():
    """hv_swap_blocks_batch_checked over 3,000 objects (two ring slots of
    descriptors), ragged and zero sizes, scattered destinations: bytes and
    digests equal the oracle's; read_errors 0."""
    from paper_2602_00328_b200 import _native as N
    rng = np.random.default_rng(9)
    n = 3000
    sizes = rng.integers(0, 9000, n).astype(np.int64)
    sizes[::97] = 0
    offs = np.concatenate([[0], np.cumsum((sizes + 15) // 16 * 16)[:-1]]).astype(np.uint64)
    total = int(offs[-1] + sizes[-1] + 16)
    src_buf = torch.empty(total, dtype=torch.uint8, device="cuda")
    seeds = [O.stable_hash64("many", i) for i in range(n)]
    from paper_2602_00328_b200 import fetch as F
    F.fill_content(F.ptrs_tensor([src_buf.data_ptr() + int(o) for o in offs], "cuda"),
                   F.ptrs_tensor(sizes.tolist(), "cuda"), seeds)
    perm = rng.permutation(n)
    dst_buf = torch.zeros(total, dtype=torch.uint8, device="cuda")
    src = np.array([src_buf.data_ptr() + int(o) for o in offs], dtype=np.uint64)
    dst = np.array([dst_buf.data_ptr() + int(offs[p]) for p in perm], dtype=np.uint64)   # scattered
    sz = sizes.astype(np.uint64)
    # object i lands where object perm[i] started; sizes must fit: use the max slot
    fit = np.array([sizes[i] <= (int(offs[perm[i] + 1]) - int(offs[perm[i]]) if perm[i] + 1 < n else 1 << 30)
                    for i in range(n)])
    sz = np.where(fit, sz, 0).astype(np.uint64)
    exp = np.array([O.content_digest(seeds[i], int(sz[i])) for i in range(n)], dtype=np.uint64)
    scratch = torch.zeros(n, dtype=torch.int64, device="cuda")
    flags = torch.zeros(n, dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int64, device="cuda")
    N.call("hv_swap_blocks_batch_checked", src.ctypes.data, dst.ctypes.data, sz.ctypes.data, exp.ctypes.data, n,
           N.ENGINES["ldg"], 0, scratch.data_ptr(), flags.data_ptr(), err.data_ptr(), 0)
    torch.cuda.synchronize()
    assert int(err.item()) == 0 and int(flags.sum().item()) == 0
    got = dst_buf.cpu().numpy()
    for i in rng.choice(n, 200, replace=False):
        d = int(dst[i]) - dst_buf.data_ptr()
        assert np.array_equal(got[d:d + int(sz[i])], O.content(seeds[i], int(sz[i]))), i
