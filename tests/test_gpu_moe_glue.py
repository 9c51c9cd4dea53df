"""The decode glue around K4: hv_moe_route (router logits, top-k, softmax,
routed pairs sorted by expert) and hv_moe_combine (fixed-order top-k combine
plus the bf16 residual), against plain PyTorch references of the same ops.

Integer outputs (the chosen experts, counts, offsets, the stable pair order)
are exact; logits within 1e-4 of an fp64 reference (fp32 accumulation over
H <= 4096 bf16 products); probabilities within 1e-6; the combine within one
bf16 rounding of an fp32 reference."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _route(h, router, k):
    from paper_2602_00328_b200 import _native as N
    T, H = h.shape
    E = router.shape[0]
    logits = torch.full((T * E,), float("nan"), device="cuda")
    probs = torch.empty(T, k, device="cuda")
    topi = torch.empty(T, k, dtype=torch.int64, device="cuda")
    counts = torch.empty(E, dtype=torch.int32, device="cuda")
    offs = torch.empty(E, dtype=torch.int32, device="cuda")
    tok = torch.full((T * k,), -1, dtype=torch.int32, device="cuda")
    pos = torch.full((T * k,), -1, dtype=torch.int64, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("hv_moe_route", h.data_ptr(), router.data_ptr(), T, H, E, k, logits.data_ptr(), probs.data_ptr(),
           topi.data_ptr(), counts.data_ptr(), offs.data_ptr(), tok.data_ptr(), pos.data_ptr(), ticket.data_ptr(),
           0, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert int(ticket.item()) == 0                  # re-armed for the next launch
    return logits.view(T, E), probs, topi, counts, offs, tok, pos


@pytest.mark.parametrize("T,H,E,k", [(32, 2048, 60, 4), (1, 4096, 16, 2), (64, 4096, 16, 2), (5, 256, 8, 2),
                                     (256, 512, 256, 8), (7, 128, 3, 3)])
def test_route_matches_torch(T, H, E, k):
    g = torch.Generator().manual_seed(T * 1000 + E)
    h = (torch.randn(T, H, generator=g) * 0.5).to(torch.bfloat16).cuda()
    router = (torch.randn(E, H, generator=g) / H ** 0.5).to(torch.bfloat16).cuda()
    logits, probs, topi, counts, offs, tok, pos = _route(h, router, k)
    ref = (h.double() @ router.double().t())
    assert (logits.double() - ref).abs().max().item() <= 1e-4
    # chosen experts: the top-k of the kernel's own logits, largest first,
    # ties to the lower id -- and equal to fp64's wherever fp64 has no near tie
    srt = torch.sort(ref, dim=1, descending=True, stable=True)
    gap = (srt.values[:, k - 1] - srt.values[:, k]) if k < E else torch.full((T,), 1.0, dtype=ref.dtype,
                                                                                 device=ref.device)
    clear = gap > 1e-3
    assert torch.equal(topi[clear].cpu(), srt.indices[clear, :k].cpu())
    own = torch.sort(logits.cpu() * -1, dim=1, stable=True).indices[:, :k]
    assert torch.equal(topi.cpu(), own)
    top = torch.gather(logits.cpu().double(), 1, topi.cpu())
    assert (probs.cpu().double() - torch.softmax(top, dim=1)).abs().max().item() <= 1e-6
    # routed pairs, exactly as torch's stable argsort of the expert ids
    flat = topi.reshape(-1).cpu()
    order = torch.argsort(flat, stable=True)
    cnt = torch.bincount(flat, minlength=E).to(torch.int32)
    assert torch.equal(counts.cpu(), cnt)
    assert torch.equal(offs.cpu(), (torch.cumsum(cnt, 0) - cnt).to(torch.int32))
    assert torch.equal(tok.cpu(), (order // k).to(torch.int32))
    want_pos = torch.empty_like(order)
    want_pos[order] = torch.arange(order.numel())
    assert torch.equal(pos.cpu(), want_pos)
    again = _route(h, router, k)                    # deterministic, ticket re-armed
    assert all(torch.equal(a, b) for a, b in zip(again[1:], (probs, topi, counts, offs, tok, pos)))


def test_route_ties_go_to_the_lower_expert():
    """Identical router rows give identical logits: the lower expert ids win."""
    T, H, E, k = 4, 256, 12, 3
    h = torch.randn(T, H).to(torch.bfloat16).cuda()
    row = torch.randn(1, H).to(torch.bfloat16)
    router = row.repeat(E, 1).cuda()
    _logits, probs, topi, *_ = _route(h, router, k)
    assert torch.equal(topi.cpu(), torch.arange(k).repeat(T, 1))
    assert torch.allclose(probs.cpu(), torch.full((T, k), 1.0 / k))


@pytest.mark.parametrize("T,H,k,rs", [(32, 2048, 4, 256.0), (1, 4096, 2, 1.0), (16, 256, 2, 0.5)])
def test_combine_matches_torch(T, H, k, rs):
    from paper_2602_00328_b200 import _native as N
    g = torch.Generator().manual_seed(T + H)
    P = T * k
    y = torch.randn(P, H, generator=g).cuda()
    probs = torch.softmax(torch.randn(T, k, generator=g), dim=1).cuda()
    pos = torch.randperm(P, generator=g).cuda()
    h = torch.randn(T, H, generator=g).to(torch.bfloat16).cuda()
    h0 = h.clone()
    N.call("hv_moe_combine", y.data_ptr(), probs.data_ptr(), pos.data_ptr(), h.data_ptr(), T, H, k, rs, 0,
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    s = (y[pos].view(T, k, H) * probs.unsqueeze(-1)).sum(1)
    m = s.to(torch.bfloat16)
    if rs != 1.0:
        m = (m.float() * rs).to(torch.bfloat16)
    ref = (h0.float() + m.float())
    # one bf16 rounding of the sum (fma vs separate multiply-add in fp32 may
    # flip the rounding of m), scaled by rs
    tol = (ref.abs() * 2 ** -7 + s.abs() * abs(rs) * 2 ** -7).cpu()
    assert ((h.float() - ref).abs().cpu() <= tol + 1e-6).all()


@pytest.mark.parametrize("E", [1, 16, 60, 100])
def test_stage_plan_matches_torch(E):
    """hv_moe_stage_plan against the torch formula it replaces: staged iff
    routed and host-resident; consecutive slots in expert order."""
    from paper_2602_00328_b200 import _native as N
    g = torch.Generator().manual_seed(E)
    counts = (torch.randint(0, 3, (E,), generator=g) * torch.randint(0, 2, (E,), generator=g)).to(torch.int32).cuda()
    host = (torch.rand(E, generator=g) < 0.5).cuda()
    addr = torch.randint(1 << 20, 1 << 40, (E,), generator=g).cuda()
    base, S = 1 << 32, 17_301_504
    dst, sizes, out = (torch.full((E,), -1, dtype=torch.int64, device="cuda") for _ in range(3))
    N.call("hv_moe_stage_plan", counts.data_ptr(), addr.data_ptr(), host.data_ptr(), base, S, E, dst.data_ptr(),
           sizes.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    stage = (counts > 0) & host
    rank = torch.cumsum(stage.to(torch.int64), 0) - 1
    want_dst = torch.where(stage, rank * S + base, 0)
    assert torch.equal(dst, want_dst)
    assert torch.equal(sizes, torch.where(stage, S, 0))
    assert torch.equal(out, torch.where(stage, want_dst, addr))
