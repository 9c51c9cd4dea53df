"""hv_paged_decode_attention alone, pages in local HBM (scattered), Llama-3-8B
KV shapes: config 1 (4 x 4k) and config 4 (1 x 128k).  Prints JSON: us per
layer and KV GB/s, for several split counts."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import _native as N  # noqa: E402


def run(B, ctx, splits_list, kvh=8, g=4, D=128, layers=4, balanced=()):
    """``layers`` distinct page pools are attended in turn (a decode step
    walks every layer), so the working set exceeds the 126 MB L2 and no call
    reads the previous call's pages from L2."""
    nb = ctx // 16
    n = B * nb
    page = 2 * 16 * kvh * D * 2
    layers = max(1, min(layers, (1 << 31) // (n * page)))   # <= 2 GiB of pages
    pools = [torch.empty(n, page, dtype=torch.uint8, device="cuda") for _ in range(layers)]
    for pool in pools:
        pool.view(torch.float16).normal_(0, 0.5)
    ptr_sets = [(torch.randperm(n).to("cuda") * page + pool.data_ptr()).to(torch.int64) for pool in pools]
    start = (torch.arange(B + 1, dtype=torch.int32) * nb).cuda()
    tok = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    q = torch.randn(B, kvh * g, D, device="cuda").to(torch.float16)
    out = torch.empty(B, kvh * g, D, device="cuda")
    res = {}
    cases = [(f"splits{sp}", sp, 0) for sp in splits_list]
    cases += [(f"balanced{c}", c, N.ATTN_BALANCED) for c in balanced]
    cases += [(f"balanced{c}_pdl", c, N.ATTN_BALANCED | N.ATTN_OVERLAP_PREVIOUS) for c in balanced]
    for name, sp, flags in cases:
        part = torch.empty((B * kvh * sp + (sp + B * kvh)) * g * (D + 2), device="cuda")
        s = torch.cuda.current_stream().cuda_stream

        it = [0]

        def f():
            ptrs = ptr_sets[it[0] % layers]
            it[0] += 1
            N.call("hv_paged_decode_attention_ex", ptrs.data_ptr(), start.data_ptr(), tok.data_ptr(), q.data_ptr(),
                   out.data_ptr(), part.data_ptr(), B, kvh * g, kvh, D, 16, sp, 1 / D ** 0.5, flags, s)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        res[name] = {"us": us, "GBps": n * page / (us * 1e-6) / 1e9}
    res["layers_rotated"] = layers
    return res


if __name__ == "__main__":
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    bal = (sms, 2 * sms)
    out = {"config1_4x4k": run(4, 4096, [3, 4, 5, 8], balanced=bal),
           "config4_1x128k": run(1, 131072, [18, 37], balanced=bal),
           "batch32_x_2k": run(32, 2048, [1, 2], balanced=bal)}
    print(json.dumps(out, indent=1))
