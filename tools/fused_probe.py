"""Fused expert FFN (hv_expert_ffn_gate_up/down) vs staged (K2 copy + cuBLAS
bmm) at decode shapes, with the experts resident in local HBM or in the
pinned host tier.  Prints JSON: ms per stage and weight GB/s of the
activated experts (the bytes that must cross the link)."""
import json
import os
import sys

import torch
import torch.nn.functional as TF

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import _native as N  # noqa: E402
from paper_2602_00328_b200 import fetch as F  # noqa: E402
from paper_2602_00328_b200.pool import HostTier  # noqa: E402


def timed(fn, iters=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def case(name, E, T, k, H, I, source):
    S = 3 * H * I * 2
    g = torch.Generator().manual_seed(0)
    torch.manual_seed(0)
    buf = (torch.randn(E * S // 2, device="cuda") * 0.02).to(torch.bfloat16)
    if source == "hbm":
        base, keep = buf.data_ptr(), buf
    else:
        host = HostTier(E * S)
        host.view()[:E * S] = buf.view(torch.uint8).cpu().numpy()
        del buf
        base, keep = host.device_address(), host
    h = torch.randn(T, H, generator=g).to(torch.bfloat16).cuda()
    logits = torch.randn(T, E, generator=g).cuda()
    topv, topi = logits.topk(k, dim=1)
    probs = torch.softmax(topv, dim=1)
    flat = topi.reshape(-1)
    order = torch.argsort(flat, stable=True)
    counts = torch.zeros(E, dtype=torch.int32, device="cuda").scatter_add_(0, flat,
                                                                          torch.ones_like(flat, dtype=torch.int32))
    offs = torch.cumsum(counts, 0, dtype=torch.int32) - counts
    tok = torch.div(order, k, rounding_mode="floor").to(torch.int32)
    P = flat.numel()
    addr = torch.tensor([base + e * S for e in range(E)], dtype=torch.int64, device="cuda")
    act = torch.empty(P, I, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(P, H, dtype=torch.float32, device="cuda")
    active = int((counts > 0).sum())
    wbytes = active * S
    s = torch.cuda.current_stream().cuda_stream

    # --tiled: the experts read as HV_FFN_TILED (random bytes either way, so
    # the timing needs no re-layout; tests/test_gpu_decode.py checks the bits)
    tiled = N.FFN_TILED if "--tiled" in sys.argv else 0

    def gate_up():
        N.call("hv_expert_ffn_gate_up_ex", addr.data_ptr(), counts.data_ptr(), offs.data_ptr(), tok.data_ptr(),
               h.data_ptr(), act.data_ptr(), E, H, I, tiled, s)

    pdl = (N.FFN_OVERLAP_PREVIOUS if "--pdl" in sys.argv else 0) | tiled

    def down():
        N.call("hv_expert_ffn_down_ex", addr.data_ptr(), counts.data_ptr(), offs.data_ptr(), act.data_ptr(),
               y.data_ptr(), E, H, I, pdl, s)

    def fused():
        gate_up()
        down()

    # staged: K2 fetch of the active experts into compact slots, then dense bmm
    ex = torch.nonzero(counts > 0).flatten().tolist()
    stage = torch.empty(len(ex), S, dtype=torch.uint8, device="cuda")
    sp = F.ptrs_tensor([base + e * S for e in ex], "cuda")
    dp = F.ptrs_tensor([stage.data_ptr() + i * S for i in range(len(ex))], "cuda")
    sz = F.ptrs_tensor([S] * len(ex), "cuda")
    K = len(ex)
    w = stage.view(torch.bfloat16).view(K, 3 * I * H)
    gate, up, dn = w[:, :I * H].view(K, I, H), w[:, I * H:2 * I * H].view(K, I, H), w[:, 2 * I * H:].view(K, H, I)

    def staged():
        F.batch_copy(sp, dp, sz, stream=s)
        x = h.unsqueeze(0).expand(K, T, H)
        a = TF.silu(torch.bmm(x, gate.transpose(1, 2))) * torch.bmm(x, up.transpose(1, 2))
        return torch.bmm(a, dn.transpose(1, 2)).sum(0)

    r = {"experts_active": active, "routed_pairs": P, "weight_bytes": wbytes}
    for nm, fn in (("fused", fused), ("fused_gate_up", gate_up), ("fused_down", down), ("staged", staged)):
        ms = timed(fn, iters=10 if source == "hbm" else 3)
        r[nm] = {"ms": ms, "weight_GBps": wbytes * (2 / 3 if nm == "fused_gate_up" else 1 / 3 if nm == "fused_down"
                                                    else 1) / (ms * 1e-3) / 1e9}
    r["speedup_fused_vs_staged"] = r["staged"]["ms"] / r["fused"]["ms"]
    if isinstance(keep, HostTier):
        keep.close()
    del keep
    return r


def main():
    out = {}
    srcs = [a for a in sys.argv[1:] if a in ("hbm", "host")] or ["hbm", "host"]
    for src in srcs:
        shapes = [("qwen_b32", 60, 32, 4, 2048, 1408), ("phi_b1", 16, 1, 2, 4096, 6400),
                  ("phi_b16", 16, 16, 2, 4096, 6400), ("phi_b64", 16, 64, 2, 4096, 6400)]
        if "swapped" in sys.argv:   # H and I exchanged: gate/up get K = 1,408, down K = 2,048
            shapes = [("qwen_b32", 60, 32, 4, 2048, 1408), ("qwen_b32_swapped", 60, 32, 4, 1408, 2048)]
        for name, E, T, k, H, I in shapes:
            out[f"{name}_{src}"] = case(name, E, T, k, H, I, src)
            torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
