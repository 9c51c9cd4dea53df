"""The fetch path with the donor on another GPU (NVLink P2P), the tier the
north star names.  Every test is parametrized over the donor device: "self"
(the donor pool on the compute GPU, runs on any box) and "peer" (device 1;
skipped unless a second GPU is visible).  The bodies are identical, so the
single-GPU run checks the test logic and a multi-GPU box checks SM-issued
loads, the TMA bulk engine and the copy engine on a real peer VA, bit-exact
against the oracle.  A 2-process NCCL check of the collectives bench.py
issues at N>1 runs when two GPUs exist."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import harvest_oracle as O

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DONORS = ["self", pytest.param("peer", marks=pytest.mark.skipif(
    not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs a second GPU"))]


def _donor(kind):
    return 0 if kind == "self" else 1


def _u64(vals):
    return torch.tensor(np.asarray(vals, dtype=np.uint64).view(np.int64), device="cuda:0")


def _placed_experts(donor, sizes, tag="pd"):
    """A system on cuda:0 whose pool lives on `donor`; objects of `sizes`
    written to the host tier by the oracle, placed with harvest_alloc and
    copied in (K3) -- the rebalance path."""
    from paper_2602_00328_b200.memalloc import Segment
    from paper_2602_00328_b200.runtime import AllocationHints
    from paper_2602_00328_b200.system import HarvestSystem
    total = sum(sizes)
    sysm = HarvestSystem(0, donors=[donor], donor_bytes=total + (64 << 20), host_bytes=total, local_bytes=total)
    rt, off, seeds, handles, offs = sysm.runtime, 0, [], [], []
    for i, s in enumerate(sizes):
        sd = O.expert_seed(tag, 0, i)
        O.fill_batch([sysm.host.host_address(off)], [s], [sd])
        h = rt.harvest_alloc(s, AllocationHints(client_id=tag))
        assert h is not None and h.device_id == 1
        rt.app_transfer(src=(sysm.host_id, Segment(off, s)), dst=(h.device_id, Segment(h.base, s)), size=s,
                        tag=(tag, i), handle=h, payload=sd)
        seeds.append(sd)
        handles.append(h)
        offs.append(off)
        off += s
    sysm.loop.run()
    sysm.engine.synchronize()
    return sysm, seeds, handles, offs


SIZES = [17_301_504, 1 << 20, 4096 + 16, 65536, 3 * (1 << 20) + 8, 17_301_504]


@pytest.mark.parametrize("donor", DONORS)
@pytest.mark.parametrize("engine", ["ldg", "ldg16", "tma", "ldg+il", "auto"])
def test_expert_fetch_from_donor_bit_exact(donor, engine):
    """K2 (and the engine per source) reading a donor pool: every object's
    digest equals the oracle's."""
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200 import _native as N
    sysm, seeds, handles, _ = _placed_experts(_donor(donor), SIZES)
    rt = sysm.runtime
    src = np.array([rt.address(h) for h in handles], dtype=np.uint64)
    dst_buf = torch.empty(sum(SIZES), dtype=torch.uint8, device="cuda:0")
    dst = np.array([dst_buf.data_ptr() + int(o) for o in np.cumsum([0] + SIZES[:-1])], dtype=np.uint64)
    sz = np.array(SIZES, dtype=np.uint64)
    N.call("hv_swap_blocks_batch", src.ctypes.data, dst.ctypes.data, sz.ctypes.data, len(SIZES),
           N.ENGINES[engine], 0, sysm.engine.stream)
    sysm.engine.synchronize()
    dg = F.digest(_u64(dst), _u64(sz)).cpu().numpy().view(np.uint64)
    for i, (sd, s) in enumerate(zip(seeds, SIZES)):
        assert int(dg[i]) == O.content_digest(sd, s), (engine, i)
    sysm.close()


@pytest.mark.parametrize("donor", DONORS)
def test_checked_fetch_and_copy_engine_from_donor(donor):
    """The fused fetch + content check (read_errors, moe.py:315-319) and the
    copy engine (cudaMemcpyAsync, the baseline of PAPER.md:200) on the
    donor's VA; one injected corruption on the donor is counted once."""
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200 import _native as N
    sysm, seeds, handles, _ = _placed_experts(_donor(donor), SIZES, tag="pc")
    rt = sysm.runtime
    n = len(SIZES)
    src = np.array([rt.address(h) for h in handles], dtype=np.uint64)
    sz = np.array(SIZES, dtype=np.uint64)
    exp = np.array([O.content_digest(sd, s) for sd, s in zip(seeds, SIZES)], dtype=np.uint64)
    dst_buf = torch.empty(sum(SIZES), dtype=torch.uint8, device="cuda:0")
    dst = np.array([dst_buf.data_ptr() + int(o) for o in np.cumsum([0] + SIZES[:-1])], dtype=np.uint64)
    scratch = torch.zeros(n, dtype=torch.int64, device="cuda:0")
    errors = torch.zeros(1, dtype=torch.int64, device="cuda:0")
    N.call("hv_swap_blocks_batch_checked", src.ctypes.data, dst.ctypes.data, sz.ctypes.data, exp.ctypes.data, n,
           N.ENGINE_AUTO, 0, scratch.data_ptr(), 0, errors.data_ptr(), sysm.engine.stream)
    sysm.engine.synchronize()
    assert int(errors.item()) == 0
    # the copy engine on the same sources
    dst_buf.zero_()
    F.ce_batch_copy(src, dst, sz, batched=True)
    torch.cuda.synchronize()
    dg = F.digest(_u64(dst), _u64(sz)).cpu().numpy().view(np.uint64)
    assert np.array_equal(dg, exp)
    # corrupt one byte of object 2 where it lies on the donor
    flip = np.array([O.content(seeds[2], 101)[100] ^ 0xFF], dtype=np.uint8)
    N.call("hv_memcpy_h2d", int(src[2]) + 100, flip.ctypes.data, 1, None)
    torch.cuda.synchronize()
    N.call("hv_swap_blocks_batch_checked", src.ctypes.data, dst.ctypes.data, sz.ctypes.data, exp.ctypes.data, n,
           N.ENGINE_AUTO, 0, scratch.data_ptr(), 0, errors.data_ptr(), sysm.engine.stream)
    sysm.engine.synchronize()
    assert int(errors.item()) == 1
    sysm.close()


@pytest.mark.parametrize("donor", DONORS)
def test_kv_pages_on_donor_gather_and_attention_in_place(donor):
    """KV blocks evicted to slabs in the donor's pool: every page gathered by
    K1 equals the oracle's content, and decode attention reading the pages in
    place (K5 over the donor VA) equals the all-local run bit for bit."""
    from paper_2602_00328_b200.kv import KVCacheManager, KVModelSpec, KVTier
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    from paper_2602_00328_b200.runtime import Durability
    from paper_2602_00328_b200.system import HarvestSystem
    m = KVModelSpec("tiny", num_layers=4, kv_heads=2, head_dim=64)
    nblk = 48
    sysm = HarvestSystem(0, donors=[_donor(donor)], donor_bytes=8 * 8 * m.block_bytes, host_bytes=1 << 20,
                         local_bytes=1 << 20)
    kv = KVCacheManager(sysm, m, local_blocks=nblk, host_blocks=64, slab_blocks=8, durability=Durability.LOSSY,
                        content="fp16")
    for s in range(3):
        kv.append_kv(s, 16 * 16)
    seqs = [0, 1, 2]
    ref = KVAttentionDecoder(kv, seqs, q_heads=4, seed=3).step().clone()
    kv.evict(nblk * m.block_bytes)
    assert all(b.tier == KVTier.PEER_HBM for b in kv.table.values())
    ids = sorted(kv.table)
    dst = torch.empty(len(ids) * m.page_bytes, dtype=torch.uint8, device="cuda:0")
    for layer in range(m.num_layers):
        kv.gather_layer(layer, ids, dst)
        kv.sys.engine.synchronize()
        got = dst.cpu().numpy().reshape(len(ids), m.page_bytes)
        for i, bid in enumerate(ids):
            b = kv.table[bid]
            want = O.weights(O.kv_seed(layer, b.sequence_id, b.index), m.page_bytes)   # content="fp16"
            assert np.array_equal(got[i], want), (bid, layer)
    for fused in (False, True):
        out = KVAttentionDecoder(kv, seqs, q_heads=4, seed=3, fused=fused).step()
        torch.cuda.synchronize()
        assert torch.equal(out, ref), fused
    sysm.loop.run()
    kv.close()
    sysm.close()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_nccl_rank_group_two_gpus():
    """The collectives bench.py issues at N>1 (RankGroup over NCCL: handle
    all_gather, decide, max, any, barrier) on two GPUs, one process each."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29561",
                        os.path.join(REPO, "tools", "nccl_rankgroup_smoke.py")],
                       capture_output=True, text=True, timeout=300, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.count('"ok": true') == 2, r.stdout
