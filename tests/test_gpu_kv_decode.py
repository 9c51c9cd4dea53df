"""Decode attention over a tiered paged KV cache (kv_decode.KVAttentionDecoder):
per-layer K1 gathers from local / peer / host pages overlapped with GQA
attention.  Outputs must be bit-identical to the same decoder over an
all-local cache, survive revocation, and match an fp32 reference computed
from the oracle's page content (tolerance stated below)."""
import numpy as np
import pytest
import torch

from oracle import harvest_oracle as O

pytestmark = pytest.mark.gpu


def _model():
    from paper_2602_00328_b200.kv import KVModelSpec
    return KVModelSpec("tiny-kv", num_layers=3, kv_heads=2, head_dim=64)


def _cache(local_blocks, donor_slabs, durability="BACKED", seqs=2, tokens=50, lengths=None):
    from paper_2602_00328_b200.kv import KVCacheManager
    from paper_2602_00328_b200.runtime import Durability
    from paper_2602_00328_b200.system import HarvestSystem
    m = _model()
    slab_blocks = 2
    sysm = HarvestSystem(0, donors=[0] if donor_slabs else [], donor_bytes=max(1, donor_slabs) * slab_blocks * m.block_bytes,
                         host_bytes=1 << 20, local_bytes=1 << 20)
    kv = KVCacheManager(sysm, m, local_blocks, host_blocks=64, slab_blocks=slab_blocks,
                        durability=Durability[durability], content="fp16")
    for s in range(seqs):
        kv.append_kv(s, lengths[s] if lengths else tokens)
    return sysm, kv, m


def _reference(kv, m, dec):
    """fp32 attention from the oracle's page bytes (fp16 KV)."""
    out = torch.empty(dec.L, dec.B, dec.Hq, m.head_dim)
    for layer in range(m.num_layers):
        for bi, s in enumerate(dec.seqs):
            pages = [O.weights(O.kv_seed(layer, s, kv.table[bid].index), m.page_bytes)
                     for bid in kv.seq_blocks[s]]
            a = torch.from_numpy(np.concatenate(pages).view(np.float16).astype(np.float32))
            a = a.view(len(pages), 2, m.block_tokens, m.kv_heads, m.head_dim)
            k = a[:, 0].reshape(-1, m.kv_heads, m.head_dim)[:dec.tokens[bi]]
            v = a[:, 1].reshape(-1, m.kv_heads, m.head_dim)[:dec.tokens[bi]]
            q = dec.q[layer, bi].float().cpu()                             # [Hq, D]
            g = dec.Hq // m.kv_heads
            kk = k.repeat_interleave(g, dim=1).transpose(0, 1)             # [Hq, T, D]
            vv = v.repeat_interleave(g, dim=1).transpose(0, 1)
            w = torch.softmax((kk @ q.unsqueeze(-1)).squeeze(-1) / m.head_dim ** 0.5, dim=-1)
            out[layer, bi] = (w.unsqueeze(-1) * vv).sum(1)
    return out


def test_tiered_kv_decode_equals_all_local_and_fp32():
    from paper_2602_00328_b200.kv import KVTier
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    from tests.refcheck import verify_release_ordering
    sysm, kv, m = _cache(local_blocks=4, donor_slabs=1)
    tiers = {b.tier for b in kv.table.values()}
    assert KVTier.PEER_HBM in tiers and KVTier.HOST_DRAM in tiers and KVTier.LOCAL_HBM in tiers
    dec = KVAttentionDecoder(kv, [0, 1], q_heads=4, seed=3)
    assert dec.T == 50
    out = dec.step()
    out2 = dec.step()
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    lsys, lkv, _ = _cache(local_blocks=16, donor_slabs=0)
    assert all(b.tier == KVTier.LOCAL_HBM for b in lkv.table.values())
    ldec = KVAttentionDecoder(lkv, [0, 1], q_heads=4, seed=3)
    ref_local = ldec.step()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref_local.view(torch.int16))      # bit-identical
    ref = _reference(kv, m, dec)
    err = (out.float().cpu() - ref).abs().max().item()
    # fp16 KV / queries, fp32 softmax reference: |err| <= 2e-2 (outputs are O(1))
    assert err <= 2e-2, err
    sysm.loop.run()
    assert verify_release_ordering(sysm.loop.log) == []
    kv.close(); sysm.close(); lkv.close(); lsys.close()


@pytest.mark.parametrize("durability", ["BACKED", "LOSSY"])
def test_kv_decode_survives_revocation(durability):
    """Every peer slab revoked between steps: Backed blocks are read from host,
    Lossy ones are recomputed; outputs stay bit-identical."""
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    from paper_2602_00328_b200.runtime import RevokeReason
    from tests.refcheck import verify_release_ordering
    sysm, kv, m = _cache(local_blocks=4, donor_slabs=2, durability=durability)
    dec = KVAttentionDecoder(kv, [0, 1], q_heads=4, seed=5)
    first = dec.step().clone()
    for s in kv.slabs:
        if s.live:
            sysm.runtime.revoke(s.handle, RevokeReason.EXTERNAL_RECLAIM)
    sysm.loop.run()                        # drains wait for the step's gathers
    assert not any(s.live for s in kv.slabs)
    again = dec.step()
    torch.cuda.synchronize()
    assert torch.equal(first.view(torch.int16), again.view(torch.int16))
    sysm.loop.run()
    assert verify_release_ordering(sysm.loop.log) == []
    kv.close(); sysm.close()


@pytest.mark.parametrize("D,kvh,g", [(128, 2, 4), (64, 2, 2), (128, 8, 4), (64, 1, 8), (128, 1, 8), (128, 4, 1)])
@pytest.mark.parametrize("splits", [1, 3, 64])
def test_paged_attention_kernel_matches_fp32(D, kvh, g, splits):
    """hv_paged_decode_attention on scattered pages: ragged sequence lengths
    (partial last blocks, a one-block sequence), any split count.  fp16 K/V/q,
    fp32 reference: |err| <= 2e-3 (outputs are O(1))."""
    from paper_2602_00328_b200 import _native as N
    torch.manual_seed(D + kvh + g)
    tokens = [37, 16, 100]
    nblk = [(t + 15) // 16 for t in tokens]
    n = sum(nblk)
    page_elems = 2 * 16 * kvh * D
    pool = (torch.randn(n + 5, page_elems, device="cuda") * 0.5).to(torch.float16)
    slots = torch.randperm(n + 5)[:n]
    ptrs = torch.tensor([pool[int(s)].data_ptr() for s in slots], dtype=torch.int64, device="cuda")
    start = torch.tensor([0] + list(np.cumsum(nblk)), dtype=torch.int32, device="cuda")
    tok = torch.tensor(tokens, dtype=torch.int32, device="cuda")
    B, Hq = len(tokens), kvh * g
    q = torch.randn(B, Hq, D, device="cuda").to(torch.float16)
    out = torch.full((B, Hq, D), float("nan"), device="cuda")
    part = torch.empty(B * kvh * splits * g * (D + 2), device="cuda")
    scale = 1.0 / D ** 0.5
    N.call("hv_paged_decode_attention", ptrs.data_ptr(), start.data_ptr(), tok.data_ptr(), q.data_ptr(),
           out.data_ptr(), part.data_ptr(), B, Hq, kvh, D, 16, splits, scale, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for b in range(B):
        pages = pool[slots[int(start[b]):int(start[b + 1])]].float().view(-1, 2, 16, kvh, D)
        k = pages[:, 0].reshape(-1, kvh, D)[:tokens[b]].transpose(0, 1).repeat_interleave(g, dim=0)  # [Hq, T, D]
        v = pages[:, 1].reshape(-1, kvh, D)[:tokens[b]].transpose(0, 1).repeat_interleave(g, dim=0)
        w = torch.softmax((k @ q[b].float().unsqueeze(-1)).squeeze(-1) * scale, dim=-1)
        ref = (w.unsqueeze(-1) * v).sum(1)
        assert (out[b] - ref).abs().max().item() <= 2e-3, (b, (out[b] - ref).abs().max().item())


def test_fused_in_place_equals_gathered():
    """fused=True (attention over the pages where they lie, no K1) gives the
    same bits as the gathered mode; both read peer, host and local pages."""
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    from tests.refcheck import verify_release_ordering
    sysm, kv, m = _cache(local_blocks=4, donor_slabs=1)
    a = KVAttentionDecoder(kv, [0, 1], q_heads=4, seed=7).step()
    b = KVAttentionDecoder(kv, [0, 1], q_heads=4, seed=7, fused=True).step()
    c = KVAttentionDecoder(kv, [0, 1], q_heads=4, seed=7, fused=True, splits=1).step()
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert (a - c).abs().max().item() <= 1e-5          # another split count: same math, other order
    sysm.loop.run()
    assert verify_release_ordering(sysm.loop.log) == []
    kv.close(); sysm.close()


def test_ragged_batch_in_place_matches_fp32():
    """Sequences of different lengths in one batch (per-sequence block ranges
    and token counts), pages spread over local, peer and host."""
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    sysm, kv, m = _cache(local_blocks=4, donor_slabs=1, seqs=3, lengths=[50, 17, 96])
    dec = KVAttentionDecoder(kv, [0, 1, 2], q_heads=4, seed=9, fused=True)
    assert dec.tokens == [50, 17, 96]
    out = dec.step()
    gat = KVAttentionDecoder(kv, [0, 1, 2], q_heads=4, seed=9).step()
    torch.cuda.synchronize()
    assert torch.equal(out, gat)
    ref = _reference(kv, m, dec)
    assert (out.float().cpu() - ref).abs().max().item() <= 2e-2
    sysm.loop.run()
    kv.close(); sysm.close()


@pytest.mark.parametrize("fused", [False, True])
def test_graph_replay_equals_eager_across_revocation(fused):
    """capture_graph(): a step is one table upload plus one CUDA graph replay
    (broadcast, K1 gathers, K5 attention on two streams).  Revoking every
    slab between replays re-points the uploaded table at the host copies;
    outputs stay bit-identical to eager steps, and drains wait for replays."""
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    from paper_2602_00328_b200.runtime import RevokeReason
    from tests.refcheck import verify_release_ordering
    sysm, kv, m = _cache(local_blocks=4, donor_slabs=1)
    eager = KVAttentionDecoder(kv, [0, 1], q_heads=4, seed=4, fused=fused).step().clone()
    dec = KVAttentionDecoder(kv, [0, 1], q_heads=4, seed=4, fused=fused)
    dec.capture_graph()
    assert torch.equal(dec.step(), eager)
    for s in kv.slabs:
        if s.live:
            sysm.runtime.revoke(s.handle, RevokeReason.EXTERNAL_RECLAIM)
    sysm.loop.run()
    again = dec.step().clone()
    torch.cuda.synchronize()
    assert torch.equal(again, eager)
    sysm.loop.run()
    assert verify_release_ordering(sysm.loop.log) == []
    kv.close(); sysm.close()


@pytest.mark.parametrize("durability", ["BACKED", "LOSSY"])
def test_kv_revocation_completes_while_steps_stream(durability):
    """Decode steps back to back with a revocation issued between them: the
    next step drains the slab (no host sync by the caller), later steps read
    the host copy / recompute, and the outputs do not change."""
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    from paper_2602_00328_b200.runtime import RevokeReason
    sysm, kv, m = _cache(local_blocks=4, donor_slabs=2, durability=durability)
    dec = KVAttentionDecoder(kv, [0, 1], q_heads=4, seed=2, fused=True)
    first = dec.step().clone()
    live = [s for s in kv.slabs if s.live]
    for s in live:
        sysm.runtime.revoke(s.handle, RevokeReason.EXTERNAL_RECLAIM)
    for _ in range(3):
        out = dec.step()
    assert all(sysm.runtime.lookup(s.handle) is None for s in live)
    torch.cuda.synchronize()
    assert torch.equal(out, first)
    kv.close(); sysm.close()


@pytest.mark.parametrize("splits", [1, 3, 64])
def test_trailing_blocks_past_token_count(splits):
    """a page table may list more blocks than a sequence's token
    count covers (KVAttentionDecoder(tokens=...) keeps every block).  Blocks
    past the tokens are neither read nor allowed to poison the softmax: with
    several splits a warp's first block can be fully masked, which used to
    give exp(-inf - -inf) = NaN.  A zero-token sequence yields zeros."""
    from paper_2602_00328_b200 import _native as N
    torch.manual_seed(11)
    D, kvh, g = 128, 2, 4
    tokens = [37, 5, 100, 0]
    nblk = [8, 6, 10, 3]                       # far more blocks than the tokens need
    n = sum(nblk)
    pool = (torch.randn(n, 2 * 16 * kvh * D, device="cuda") * 0.5).to(torch.float16)
    pool[torch.isnan(pool)] = 0
    ptrs = torch.tensor([pool[i].data_ptr() for i in range(n)], dtype=torch.int64, device="cuda")
    start = torch.tensor([0] + list(np.cumsum(nblk)), dtype=torch.int32, device="cuda")
    tok = torch.tensor(tokens, dtype=torch.int32, device="cuda")
    B, Hq = len(tokens), kvh * g
    q = torch.randn(B, Hq, D, device="cuda").to(torch.float16)
    out = torch.full((B, Hq, D), float("nan"), device="cuda")
    part = torch.empty(B * kvh * splits * g * (D + 2), device="cuda")
    scale = 1.0 / D ** 0.5
    N.call("hv_paged_decode_attention", ptrs.data_ptr(), start.data_ptr(), tok.data_ptr(), q.data_ptr(),
           out.data_ptr(), part.data_ptr(), B, Hq, kvh, D, 16, splits, scale, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    for b in range(B):
        if tokens[b] == 0:
            assert (out[b] == 0).all()
            continue
        pages = pool[int(start[b]):int(start[b + 1])].float().view(-1, 2, 16, kvh, D)
        k = pages[:, 0].reshape(-1, kvh, D)[:tokens[b]].transpose(0, 1).repeat_interleave(g, dim=0)
        v = pages[:, 1].reshape(-1, kvh, D)[:tokens[b]].transpose(0, 1).repeat_interleave(g, dim=0)
        w = torch.softmax((k @ q[b].float().unsqueeze(-1)).squeeze(-1) * scale, dim=-1)
        ref = (w.unsqueeze(-1) * v).sum(1)
        assert (out[b] - ref).abs().max().item() <= 2e-3


@pytest.mark.parametrize("fused", [False, True])
def test_decoder_with_tokens_shorter_than_sequences(fused):
    """KVAttentionDecoder(tokens=20) over 96-token sequences: finite, equal
    to the fp32 reference over the first 20 tokens, at several splits."""
    from paper_2602_00328_b200.kv_decode import KVAttentionDecoder
    sysm, kv, m = _cache(local_blocks=4, donor_slabs=1, seqs=2, tokens=96)
    outs = []
    for splits in (None, 4):
        dec = KVAttentionDecoder(kv, [0, 1], q_heads=4, tokens=20, seed=5, fused=fused, splits=splits)
        assert dec.tokens == [20, 20]
        out = dec.step()
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all()
        ref = _reference(kv, m, dec)
        assert (out.float().cpu() - ref).abs().max().item() <= 2e-2
        outs.append(out)
    sysm.loop.run()
    kv.close(); sysm.close()
