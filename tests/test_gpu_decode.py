"""MoE decode over Harvest tiers (moe._DecodeRun semantics, moe.py:211-340)
with real compute: outputs must be bit-identical to an all-local run, and
the math must match a plain PyTorch fp32 reference of the same MoE layer
stack (tolerance stated below)."""
import numpy as np
import pytest
import torch

from oracle import harvest_oracle as O

pytestmark = pytest.mark.gpu
RS = 256.0  # residual scale: makes the tiny MoE delta visible in bf16 (power of two: exact)


def _setup(model, peer_experts, microbatches=2, tokens=16, seed=0, layout="row"):
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore, rebalance
    from paper_2602_00328_b200.system import HarvestSystem
    L, E, S = model.num_layers, model.num_experts, model.expert_size
    sysm = HarvestSystem(0, donors=[0], donor_bytes=max(1, peer_experts) * S, host_bytes=L * E * S,
                         local_bytes=1 << 20)
    store = ExpertStore(model, sysm.host_id, sysm.host)
    store.fill_host(0, weights=True, layout=layout)
    res = ExpertResidency(model)
    counts = np.ones((L, E), dtype=np.int64)
    if peer_experts:
        rebalance(sysm.loop, sysm.runtime, model, res, counts, sysm.host_id, max_migrations=peer_experts, store=store)
        sysm.loop.run()
    fetcher = ExpertFetcher(sysm.runtime, model, res, store)
    dec = MoEDecoder(fetcher, tokens=tokens, microbatches=microbatches, seed=seed, residual_scale=RS)
    return sysm, store, res, fetcher, dec


def _all_local(model, tokens, microbatches, seed, host_store):
    """Same decoder with every expert LOCAL: resident weights in HBM."""
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.moe import ExpertFetcher, ExpertResidency, ExpertStore
    from paper_2602_00328_b200.system import HarvestSystem
    L, E, S = model.num_layers, model.num_experts, model.expert_size
    sysm = HarvestSystem(0, host_bytes=1, local_bytes=1)
    resident = torch.from_numpy(host_store.host.view()[:L * E * S].copy()).cuda()
    res = ExpertResidency(model)
    for layer in range(L):
        for e in range(E):
            res.set_tier(layer, e, Tier.LOCAL_HBM)
    store = ExpertStore(model, sysm.host_id, None)
    store.layout = host_store.layout          # the resident copy holds the host tier's bytes
    local_addr = [[resident.data_ptr() + (layer * E + e) * S for e in range(E)] for layer in range(L)]
    fetcher = ExpertFetcher(sysm.runtime, model, res, store, local_addr=local_addr)
    dec = MoEDecoder(fetcher, tokens=tokens, microbatches=microbatches, seed=seed, residual_scale=RS)
    return sysm, dec, resident


def _tiny():
    from paper_2602_00328_b200.moe import MoEProfile
    H, I = 256, 128
    return MoEProfile("tiny-moe", num_layers=3, num_experts=8, top_k=2, expert_size=3 * H * I * 2, hidden=H,
                      intermediate=I)


def _torch_reference(model, dec, x, steps):
    """Plain fp32 PyTorch MoE stack (router -> top-k softmax -> SwiGLU experts),
    weights from the oracle's bf16 weight generator."""
    from paper_2602_00328_b200.moe import expert_content
    L, E, H, I = model.num_layers, model.num_experts, model.hidden, model.intermediate
    W = {}
    for layer in range(L):
        for e in range(E):
            w = torch.from_numpy(O.weights(expert_content(model, layer, e), model.expert_size).view(np.int16).copy())
            w = w.view(torch.bfloat16).float()
            W[layer, e] = (w[:I * H].view(I, H), w[I * H:2 * I * H].view(I, H), w[2 * I * H:].view(H, I))
    h = x.float().cpu()
    for _ in range(steps):
        for layer in range(L):
            r = dec.router[layer].float().cpu()
            logits = h @ r.t()
            topv, topi = logits.topk(model.top_k, dim=1)
            p = torch.softmax(topv, dim=1)
            out = torch.zeros_like(h)
            for t in range(h.shape[0]):
                for j in range(model.top_k):
                    g, u, d = W[layer, int(topi[t, j])]
                    out[t] += p[t, j] * (d @ (torch.nn.functional.silu(g @ h[t]) * (u @ h[t])))
            h = h + RS * out
    return h


@pytest.mark.parametrize("microbatches", [1, 2])
def test_decode_offloaded_equals_all_local(microbatches):
    model = _tiny()
    L, E = model.num_layers, model.num_experts
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=L * E // 2, microbatches=microbatches)
    from paper_2602_00328_b200.memalloc import Tier
    tiers = [e.tier for e in res.entries.values()]
    assert tiers.count(Tier.PEER_HBM) == L * E // 2 and tiers.count(Tier.HOST_DRAM) == L * E // 2
    out = dec.decode(3)
    torch.cuda.synchronize()
    sys2, dec2, _keep = _all_local(model, 16, microbatches, 0, store)
    out2 = dec2.decode(3)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), out2.view(torch.int16))   # bit-identical
    assert torch.isfinite(out.float()).all()
    sysm.loop.run()
    sysm.close()
    sys2.close()


def test_decode_matches_fp32_reference():
    model = _tiny()
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=6, microbatches=2)
    out = dec.decode(1)
    torch.cuda.synchronize()
    ref = _torch_reference(model, dec, dec.x0, 1)
    x0 = dec.x0.float().cpu()
    d_gpu, d_ref = out.float().cpu() - x0, ref - x0            # the MoE contribution of 3 layers
    scale = d_ref.abs().max().item()
    assert scale > 0.05 * x0.abs().max().item()                 # the delta is not lost in bf16 rounding
    err = (d_gpu - d_ref).abs().max().item()
    # bf16 weights/activations/residual vs fp32 math: tolerance 5e-2 of the delta scale
    assert err <= 5e-2 * scale, (err, scale)
    sysm.loop.run()
    sysm.close()


def test_decode_survives_revocation_midway():
    """Revoke every peer slab between steps: later fetches come from the host
    copy and the outputs still equal the all-local run."""
    from paper_2602_00328_b200.runtime import RevokeReason
    model = _tiny()
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=12, microbatches=2)
    h = dec.step(dec.x0)
    for hdl in list(fetcher.handles.values()):
        sysm.runtime.revoke(hdl, RevokeReason.PRESSURE)
    sysm.loop.run()                     # drain -> invalidate -> callback (residency -> host)
    assert not fetcher.handles
    dec.sync_tables()
    h = dec.step(h)
    torch.cuda.synchronize()
    sys2, dec2, _keep = _all_local(model, 16, 2, 0, store)
    h2 = dec2.step(dec2.step(dec2.x0))
    torch.cuda.synchronize()
    assert torch.equal(h.view(torch.int16), h2.view(torch.int16))
    sysm.close()
    sys2.close()


@pytest.mark.parametrize("microbatches", [1, 2])
def test_graph_replay_equals_eager_and_all_local(microbatches):
    """capture_graph(): every later step is one CUDA graph replay (router,
    device-side fetch plan, K2 fetch on the fetch stream, expert FFN).  A
    revocation between replays updates the captured address table in place;
    outputs stay bit-identical to the all-local eager run."""
    from paper_2602_00328_b200.runtime import RevokeReason
    model = _tiny()
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=12, microbatches=microbatches)
    dec.capture_graph()
    h = dec.step(dec.x0)
    h = dec.step(h)
    for hdl in list(fetcher.handles.values()):
        sysm.runtime.revoke(hdl, RevokeReason.PRESSURE)
    sysm.loop.run()                     # drain (waits on the replay's event) -> residency -> host
    assert not fetcher.handles
    h = dec.step(h)                     # version changed: in-place table update, then replay
    out = h.clone()
    torch.cuda.synchronize()
    sys2, dec2, _keep = _all_local(model, 16, microbatches, 0, store)
    out2 = dec2.decode(3)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), out2.view(torch.int16))
    from tests.refcheck import verify_release_ordering
    assert verify_release_ordering(sysm.loop.log) == []
    sysm.close()
    sys2.close()


# ---------------------------------------------------------------- fused expert FFN (csrc/hv_ffn.cu)

@pytest.mark.parametrize("H,I,counts", [(256, 128, [3, 0, 1, 8, 64, 17]), (2048, 1408, [2, 5, 0, 1, 9, 33]),
                                        (4096, 6400, [1, 0, 2])])
def test_fused_ffn_kernels_match_fp32(H, I, counts):
    """hv_expert_ffn_gate_up / hv_expert_ffn_down against fp32 torch on random
    bf16 experts, ragged token counts (0 .. 64 per expert), tokens gathered
    through an arbitrary pair -> row map.  Tolerance: act is rounded to bf16
    (rel 2^-8) and both GEMVs accumulate in fp32: |err| <= 1e-2 * max|ref|."""
    from paper_2602_00328_b200 import _native as N
    g = torch.Generator().manual_seed(H + I)
    E, T = len(counts), 64
    S = 3 * H * I * 2
    W = (torch.randn(E, 3 * H * I, generator=g) * 0.03).to(torch.bfloat16).cuda()
    x = (torch.randn(T, H, generator=g)).to(torch.bfloat16).cuda()
    cnt = torch.tensor(counts, dtype=torch.int32)
    offs = torch.cumsum(cnt, 0, dtype=torch.int32) - cnt
    P = int(cnt.sum())
    tok = torch.cat([torch.randperm(T, generator=g)[:c] for c in counts]).to(torch.int32)
    addr = torch.tensor([W[e].data_ptr() for e in range(E)], dtype=torch.int64).cuda()
    cnt_d, offs_d, tok_d = cnt.cuda(), offs.cuda(), tok.cuda()
    act = torch.full((P, I), float("nan"), dtype=torch.bfloat16, device="cuda")
    y = torch.full((P, H), float("nan"), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    N.call("hv_expert_ffn_gate_up", addr.data_ptr(), cnt_d.data_ptr(), offs_d.data_ptr(), tok_d.data_ptr(),
           x.data_ptr(), act.data_ptr(), E, H, I, s)
    N.call("hv_expert_ffn_down", addr.data_ptr(), cnt_d.data_ptr(), offs_d.data_ptr(), act.data_ptr(),
           y.data_ptr(), E, H, I, s)
    torch.cuda.synchronize()
    Wf, xf = W.float().cpu(), x.float().cpu()
    for e in range(E):
        gate, up = Wf[e, :I * H].view(I, H), Wf[e, I * H:2 * I * H].view(I, H)
        down = Wf[e, 2 * I * H:].view(H, I)
        for j in range(counts[e]):
            p = int(offs[e]) + j
            xt = xf[int(tok[p])]
            a_ref = torch.nn.functional.silu(gate @ xt) * (up @ xt)
            a_got = act[p].float().cpu()
            assert (a_got - a_ref).abs().max() <= 1e-2 * a_ref.abs().max(), (e, j)
            y_ref = down @ a_got                        # exact bf16 inputs the kernel saw
            assert (y[p].cpu() - y_ref).abs().max() <= 1e-3 * y_ref.abs().max() + 1e-6, (e, j)
    assert S == W[0].numel() * 2


@pytest.mark.parametrize("H,I,counts", [(256, 128, [3, 0, 1, 8, 64, 17]), (2048, 1408, [2, 5, 0, 1, 9, 33]),
                                        (4096, 6400, [1, 0, 2])])
def test_fused_ffn_tiled_layout_equals_row_major(H, I, counts):
    """HV_FFN_TILED: the same experts stored as swizzled 128 x 64 tiles
    (fetch.tile_expert_matrix), each tile one bulk copy on the TMA engine.
    The tiles land in shared memory byte for byte where the row-major form's
    cp.async puts them, so act and y are bitwise those of the row-major form."""
    from paper_2602_00328_b200 import _native as N
    from paper_2602_00328_b200 import fetch as F
    g = torch.Generator().manual_seed(7 + H + I)
    E, T = len(counts), 64
    W = (torch.randn(E, 3 * H * I, generator=g) * 0.03).to(torch.bfloat16).cuda()
    Wt = torch.empty_like(W)
    for e in range(E):
        Wt[e, :I * H] = F.tile_expert_matrix(W[e, :I * H].view(I, H)).reshape(-1)
        Wt[e, I * H:2 * I * H] = F.tile_expert_matrix(W[e, I * H:2 * I * H].view(I, H)).reshape(-1)
        Wt[e, 2 * I * H:] = F.tile_expert_matrix(W[e, 2 * I * H:].view(H, I)).reshape(-1)
    assert torch.equal(F.tile_expert_matrix(Wt[0, 2 * I * H:].view(H, I), inverse=True), W[0, 2 * I * H:].view(H, I))
    x = (torch.randn(T, H, generator=g)).to(torch.bfloat16).cuda()
    cnt = torch.tensor(counts, dtype=torch.int32)
    offs = torch.cumsum(cnt, 0, dtype=torch.int32) - cnt
    P = int(cnt.sum())
    tok = torch.cat([torch.randperm(T, generator=g)[:c] for c in counts]).to(torch.int32).cuda()
    cnt_d, offs_d = cnt.cuda(), offs.cuda()
    s = torch.cuda.current_stream().cuda_stream
    outs = []
    for weights, flags in ((W, 0), (Wt, N.FFN_TILED)):
        addr = torch.tensor([weights[e].data_ptr() for e in range(E)], dtype=torch.int64).cuda()
        act = torch.full((P, I), float("nan"), dtype=torch.bfloat16, device="cuda")
        y = torch.full((P, H), float("nan"), dtype=torch.float32, device="cuda")
        N.call("hv_expert_ffn_gate_up_ex", addr.data_ptr(), cnt_d.data_ptr(), offs_d.data_ptr(), tok.data_ptr(),
               x.data_ptr(), act.data_ptr(), E, H, I, flags, s)
        N.call("hv_expert_ffn_down_ex", addr.data_ptr(), cnt_d.data_ptr(), offs_d.data_ptr(), act.data_ptr(),
               y.data_ptr(), E, H, I, flags, s)
        outs.append((act, y))
    torch.cuda.synchronize()
    assert not torch.isnan(outs[0][1]).any()
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    assert torch.equal(outs[0][1].view(torch.int32), outs[1][1].view(torch.int32))


def test_fused_ffn_tiled_layout_rejects_unsupported_shapes():
    """Rows not a multiple of 128 (the mma.sync form's shapes) cannot take the
    tiled layout: refused, not silently read as row-major."""
    from paper_2602_00328_b200 import _native as N
    E, H, I = 1, 256, 192
    W = torch.zeros(E, 3 * H * I, dtype=torch.bfloat16, device="cuda")
    addr = torch.tensor([W[0].data_ptr()], dtype=torch.int64).cuda()
    one = torch.ones(1, dtype=torch.int32).cuda()
    zero = torch.zeros(1, dtype=torch.int32).cuda()
    x = torch.zeros(1, H, dtype=torch.bfloat16, device="cuda")
    act = torch.zeros(1, I, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(N.HarvestNativeError):
        N.call("hv_expert_ffn_gate_up_ex", addr.data_ptr(), one.data_ptr(), zero.data_ptr(), zero.data_ptr(),
               x.data_ptr(), act.data_ptr(), E, H, I, N.FFN_TILED, torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("microbatches", [1, 2])
def test_tiled_experts_decode_equals_row_major(microbatches):
    """Experts stored as HV_FFN_TILED tiles (ExpertStore.fill_host(layout=
    "tiled")), half on the donor and half in the host tier: the fused decoder
    (K4 in place, one bulk copy per weight tile) and the staged decoder (K2
    into the staging slots, then K4 over them) are both bit-identical to the
    fused decoder over the same logical weights stored row-major, and to the
    tiled all-local run.  The host copy's bytes are the row-major bytes
    permuted (fetch.tile_expert_matrix, inverse checked)."""
    from paper_2602_00328_b200 import fetch as F
    from paper_2602_00328_b200.decode import MoEDecoder
    model = _tiny()
    L, E, S, H, I = model.num_layers, model.num_experts, model.expert_size, model.hidden, model.intermediate
    half = L * E // 2
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=half, microbatches=microbatches)
    ref = MoEDecoder(fetcher, tokens=16, microbatches=microbatches, seed=0, residual_scale=RS, fused=True).decode(3)
    tsys, tstore, tres, tfetcher, tdec = _setup(model, peer_experts=half, microbatches=microbatches, layout="tiled")
    assert tstore.layout == "tiled" and tdec.tiled
    row = torch.from_numpy(store.host.view()[:S].copy()).view(torch.bfloat16)
    til = torch.from_numpy(tstore.host.view()[:S].copy()).view(torch.bfloat16)
    assert not torch.equal(row, til)
    assert torch.equal(F.tile_expert_matrix(til[2 * I * H:].view(H, I), inverse=True), row[2 * I * H:].view(H, I))
    fused = MoEDecoder(tfetcher, tokens=16, microbatches=microbatches, seed=0, residual_scale=RS, fused=True)
    out_f = fused.decode(3)
    out_s = tdec.decode(3)
    torch.cuda.synchronize()
    assert torch.equal(out_f.view(torch.int16), ref.view(torch.int16))
    assert torch.equal(out_s.view(torch.int16), ref.view(torch.int16))
    sys2, _d2, keep = _all_local(model, 16, microbatches, 0, tstore)
    out_l = MoEDecoder(_d2.f, tokens=16, microbatches=microbatches, seed=0, residual_scale=RS, fused=True).decode(3)
    torch.cuda.synchronize()
    assert torch.equal(out_l.view(torch.int16), ref.view(torch.int16))
    if microbatches == 1:   # host plan (copy engine for host-tier experts) over tiled experts: the same bits
        hp = MoEDecoder(tfetcher, tokens=16, microbatches=1, seed=0, residual_scale=RS, host_plan=True)
        assert torch.equal(hp.decode(3).view(torch.int16), ref.view(torch.int16))
    for s_ in (sysm, tsys):
        s_.loop.run()
    sysm.close(); tsys.close(); sys2.close()


@pytest.mark.parametrize("microbatches", [1, 2])
def test_fused_decode_offloaded_equals_all_local(microbatches):
    """fused=True reads half the experts from the donor pool and half from the
    pinned host tier in place; outputs are bit-identical to the fused all-local
    run, and within tolerance of the staged (K2 + cuBLAS) decoder."""
    from paper_2602_00328_b200.decode import MoEDecoder
    model = _tiny()
    L, E = model.num_layers, model.num_experts
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=L * E // 2, microbatches=microbatches)
    fdec = MoEDecoder(fetcher, tokens=16, microbatches=microbatches, seed=0, residual_scale=RS, fused=True)
    out = fdec.decode(3)
    staged = dec.decode(3)
    torch.cuda.synchronize()
    sys2, _dec2, keep = _all_local(model, 16, microbatches, 0, store)
    ldec = MoEDecoder(_dec2.f, tokens=16, microbatches=microbatches, seed=0, residual_scale=RS, fused=True)
    out2 = ldec.decode(3)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), out2.view(torch.int16))
    x0 = fdec.x0.float()
    d_f, d_s = out.float() - x0, staged.float() - x0
    assert (d_f - d_s).abs().max() <= 5e-2 * d_s.abs().max()
    from tests.refcheck import verify_release_ordering
    sysm.loop.run()
    assert verify_release_ordering(sysm.loop.log) == []
    sysm.close()
    sys2.close()


def test_fused_decode_matches_fp32_reference():
    from paper_2602_00328_b200.decode import MoEDecoder
    model = _tiny()
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=6, microbatches=2)
    fdec = MoEDecoder(fetcher, tokens=16, microbatches=2, seed=0, residual_scale=RS, fused=True)
    out = fdec.decode(1)
    torch.cuda.synchronize()
    ref = _torch_reference(model, fdec, fdec.x0, 1)
    x0 = fdec.x0.float().cpu()
    d_gpu, d_ref = out.float().cpu() - x0, ref - x0
    scale = d_ref.abs().max().item()
    err = (d_gpu - d_ref).abs().max().item()
    assert err <= 5e-2 * scale, (err, scale)      # same tolerance as the staged decoder
    sysm.loop.run()
    sysm.close()


def test_fused_graph_replay_with_revocation():
    """Fused step captured as one CUDA graph; revoking every peer expert between
    replays re-points the captured address table at the host copies (in place);
    outputs stay bit-identical to the fused all-local eager run, and the
    drains wait for the replays that read the revoked slabs."""
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.runtime import RevokeReason
    from tests.refcheck import verify_release_ordering
    model = _tiny()
    sysm, store, res, fetcher, _dec = _setup(model, peer_experts=12, microbatches=2)
    dec = MoEDecoder(fetcher, tokens=16, microbatches=2, seed=0, residual_scale=RS, fused=True)
    dec.capture_graph()
    h = dec.step(dec.x0)
    h = dec.step(h)
    for hdl in list(fetcher.handles.values()):
        sysm.runtime.revoke(hdl, RevokeReason.PRESSURE)
    sysm.loop.run()
    assert not fetcher.handles
    out = dec.step(h).clone()
    torch.cuda.synchronize()
    sys2, _dec2, keep = _all_local(model, 16, 2, 0, store)
    ldec = MoEDecoder(_dec2.f, tokens=16, microbatches=2, seed=0, residual_scale=RS, fused=True)
    out2 = ldec.decode(3)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), out2.view(torch.int16))
    assert verify_release_ordering(sysm.loop.log) == []
    sysm.close()
    sys2.close()


@pytest.mark.parametrize("fused", [False, True])
def test_revocation_completes_while_steps_stream(fused):
    """Steps enqueued back to back (no host sync between them) must not starve
    a revocation: the next step drains it (callbacks fire inside step()), stops
    reading the donor, and the outputs stay equal to the all-local run."""
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.runtime import RevokeReason
    from tests.refcheck import verify_release_ordering
    model = _tiny()
    sysm, store, res, fetcher, _d = _setup(model, peer_experts=12, microbatches=1)
    dec = MoEDecoder(fetcher, tokens=16, microbatches=1, seed=0, residual_scale=RS, fused=fused)
    h = dec.step(dec.x0)
    h = dec.step(h)
    revoked = list(fetcher.handles.values())
    assert revoked
    for hdl in revoked:
        sysm.runtime.revoke(hdl, RevokeReason.PRESSURE)
    for _ in range(3):                       # no loop.run()/synchronize from the test
        h = dec.step(h)
    assert not fetcher.handles               # every revocation finished inside step()
    assert all(sysm.runtime.lookup(x) is None for x in revoked)
    torch.cuda.synchronize()
    sys2, ldec0, _keep = _all_local(model, 16, 1, 0, store)
    ldec = MoEDecoder(ldec0.f, tokens=16, microbatches=1, seed=0, residual_scale=RS, fused=fused)
    out2 = ldec.decode(5)
    torch.cuda.synchronize()
    assert torch.equal(h.view(torch.int16), out2.view(torch.int16))
    sysm.loop.run()
    assert verify_release_ordering(sysm.loop.log) == []
    sysm.close()
    sys2.close()


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("tier", ["peer", "host"])
def test_offload_sweep_every_fraction_equals_all_local(tier, fused):
    """decode.offload_sweep (moe.offload_sweep, moe.py:394-415, on real
    decode): each fraction's output is bit-identical to the all-local decode
    (checked inside, raises otherwise); one row per fraction; peer handles
    are returned between fractions."""
    from paper_2602_00328_b200.decode import offload_sweep
    from paper_2602_00328_b200.memalloc import Tier
    from paper_2602_00328_b200.system import HarvestSystem
    model = _tiny()
    L, E, S = model.num_layers, model.num_experts, model.expert_size
    sysm = HarvestSystem(0, donors=[0] if tier == "peer" else [], donor_bytes=L * E * S + (4 << 20),
                         host_bytes=L * E * S, local_bytes=1 << 20)
    rows = offload_sweep(sysm, model, [0, 25, 50, 100], Tier.PEER_HBM if tier == "peer" else Tier.HOST_DRAM,
                         tokens=16, microbatches=2, fused=fused, steps=2, warmup=1)
    assert [r.fraction_pct for r in rows] == [0, 25, 50, 100]
    assert all(r.tier == tier and r.tokens_per_s > 0 for r in rows)
    assert all((r.stall_s is None) == fused for r in rows)
    if tier == "peer":                      # every peer handle went back to its donor
        assert not sysm.runtime.placement
        assert sysm.runtime.occupied_bytes(1) == 0


@pytest.mark.parametrize("microbatches", [1, 2])
def test_host_plan_decode_equals_device_plan_and_all_local(microbatches):
    """MoEDecoder(host_plan=True): each stage's plan goes back to the host and
    through the library's engine per source, so host-tier experts (1.5 MiB
    here, above the copy-engine threshold) ride the copy engine and peer ones
    the K2 kernel.  Outputs are bit-identical to the device-plan decoder and
    to the all-local run."""
    from paper_2602_00328_b200.decode import MoEDecoder
    from paper_2602_00328_b200.moe import MoEProfile
    H, I = 512, 512
    model = MoEProfile("tiny-moe-ce", num_layers=2, num_experts=8, top_k=2, expert_size=3 * H * I * 2, hidden=H,
                       intermediate=I)
    L, E = model.num_layers, model.num_experts
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=L * E // 2, microbatches=microbatches)
    hp = MoEDecoder(fetcher, tokens=16, microbatches=microbatches, seed=0, residual_scale=RS, host_plan=True)
    out = dec.decode(2)
    out_hp = hp.decode(2)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), out_hp.view(torch.int16))
    sys2, dec2, _keep = _all_local(model, 16, microbatches, 0, store)
    out2 = dec2.decode(2)
    torch.cuda.synchronize()
    assert torch.equal(out_hp.view(torch.int16), out2.view(torch.int16))
    with pytest.raises(ValueError):
        hp.capture_graph()
    sysm.loop.run()
    sysm.close()
    sys2.close()


def test_fetch_stream_is_urgent_and_node_priority_graph_equals_eager():
    """The fetch engine's stream is created at the device's greatest priority
    (a stage's fetch is dispatched ahead of the compute stream's CTAs,
    profiles/r2_priority_probe.json); a graph instantiated by the library
    with per-node priority (hv_graph_instantiate) replays bit-identically to
    torch's instantiation and to the all-local eager run."""
    import ctypes as C
    from paper_2602_00328_b200 import _native as N
    model = _tiny()
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=12, microbatches=2)
    least, greatest = C.c_int(), C.c_int()
    N.call("hv_stream_priority_range", 0, C.byref(least), C.byref(greatest))
    assert torch.cuda.ExternalStream(sysm.engine.stream).priority == greatest.value
    assert torch.cuda.ExternalStream(sysm.placement_engine.stream).priority == 0
    dec.capture_graph(node_priority=True)
    assert dec._graph_exec is not None
    h = dec.step(dec.x0)
    h = dec.step(h)
    out = dec.step(h).clone()
    torch.cuda.synchronize()
    sys2, dec2, _keep = _all_local(model, 16, 2, 0, store)
    out2 = dec2.decode(3)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), out2.view(torch.int16))
    del dec
    sysm.close()
    sys2.close()


def test_library_glue_agrees_with_torch_glue():
    """MoEDecoder.glue: the router / pair sort / combine as library kernels
    (default) or as torch ops.  Logits differ in rounding (fp32 dot vs a bf16
    GEMM), so the two agree to tolerance, and each is bit-identical to its
    own all-local run."""
    from paper_2602_00328_b200.decode import MoEDecoder
    model = _tiny()
    L, E = model.num_layers, model.num_experts
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=L * E // 2, microbatches=1)
    sys2, _d2, keep = _all_local(model, 16, 1, 0, store)
    outs = {}
    try:
        for glue in (True, False):
            MoEDecoder.glue = glue
            a = MoEDecoder(fetcher, tokens=16, microbatches=1, seed=0, residual_scale=RS, fused=True).decode(3)
            b = MoEDecoder(_d2.f, tokens=16, microbatches=1, seed=0, residual_scale=RS, fused=True).decode(3)
            torch.cuda.synchronize()
            assert torch.equal(a.view(torch.int16), b.view(torch.int16))
            outs[glue] = a
    finally:
        MoEDecoder.glue = True
    x0 = dec.x0.float()
    d_k, d_t = outs[True].float() - x0, outs[False].float() - x0
    assert (d_k - d_t).abs().max() <= 5e-2 * d_t.abs().max()
    sysm.loop.run()
    sysm.close(); sys2.close()


@pytest.mark.parametrize("layout", ["row", "tiled"])
def test_pdl_chain_changes_no_bits(layout):
    """MoEDecoder.pdl: the stage's route / K4 gate_up / K4 down / combine as a
    chain of programmatic dependent launches.  Only when kernels start
    changes, so every output bit equals the plainly launched chain's, eager
    and as a CUDA graph."""
    from paper_2602_00328_b200.decode import MoEDecoder
    model = _tiny()
    L, E = model.num_layers, model.num_experts
    sysm, store, res, fetcher, dec = _setup(model, peer_experts=L * E // 2, microbatches=1, layout=layout)
    outs = {}
    try:
        for pdl in (False, True):
            MoEDecoder.pdl = pdl
            d = MoEDecoder(fetcher, tokens=16, microbatches=1, seed=0, residual_scale=RS, fused=True)
            assert d.pdl == pdl
            eager = d.decode(3)
            d.capture_graph()
            graph = d.decode(3)
            torch.cuda.synchronize()
            assert torch.equal(eager.view(torch.int16), graph.view(torch.int16))
            outs[pdl] = eager
    finally:
        MoEDecoder.pdl = True
    assert torch.equal(outs[True].view(torch.int16), outs[False].view(torch.int16))
    sysm.loop.run()
    sysm.close()
