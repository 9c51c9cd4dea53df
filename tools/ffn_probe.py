"""Expert-FFN compute variants at decode shapes (weights already staged).
Prints JSON: ms per stage and effective weight-read GB/s."""
import json
import os
import sys

import torch
import torch.nn.functional as TF

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def t(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    out = {}
    for name, K, T, H, I in (("qwen_T32", 60, 32, 2048, 1408), ("qwen_T16", 60, 16, 2048, 1408),
                              ("phi_T1", 2, 1, 4096, 6400), ("phi_T64", 16, 64, 4096, 6400)):
        W = torch.randn(K, 3 * I * H, device="cuda", dtype=torch.bfloat16) * 0.01
        h = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        gate = W[:, :I * H].view(K, I, H)
        up = W[:, I * H:2 * I * H].view(K, I, H)
        gu = W[:, :2 * I * H].view(K, 2 * I, H)
        down = W[:, 2 * I * H:].view(K, H, I)
        wts = torch.rand(K, T, 1, device="cuda", dtype=torch.bfloat16)

        def v0():  # current: expand + 3 bmm
            x = h.unsqueeze(0).expand(K, T, H)
            a = TF.silu(torch.bmm(x, gate.transpose(1, 2))) * torch.bmm(x, up.transpose(1, 2))
            return (torch.bmm(a, down.transpose(1, 2)) * wts).sum(0)

        def v1():  # fused gate|up bmm, contiguous x
            x = h.unsqueeze(0).expand(K, T, H).contiguous()
            g = torch.bmm(x, gu.transpose(1, 2))
            a = TF.silu(g[..., :I]) * g[..., I:]
            return (torch.bmm(a, down.transpose(1, 2)) * wts).sum(0)

        def v2():  # weights as the left operand (W @ x^T): M = 2I rows per expert
            xt = h.t().unsqueeze(0).expand(K, H, T)
            g = torch.bmm(gu, xt)                       # [K, 2I, T]
            a = TF.silu(g[:, :I]) * g[:, I:]            # [K, I, T]
            y = torch.bmm(down, a)                      # [K, H, T]
            return (y * wts.transpose(1, 2)).sum(0).t()

        wbytes = K * 3 * I * H * 2
        r = {}
        for vn, fn in (("v0_3bmm", v0), ("v1_fused_gu", v1), ("v2_weights_left", v2)):
            ms = t(fn)
            r[vn] = {"ms": ms, "weight_GBps": wbytes / (ms * 1e-3) / 1e9}
        out[name] = r
        del W
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
