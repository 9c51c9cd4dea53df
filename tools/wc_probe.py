"""Pinned host tier: default (snooped) vs write-combined, for the SM-issued
fetch kernels and the copy engine.  Prints JSON."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import fetch as F  # noqa: E402
from paper_2602_00328_b200.pool import HostTier  # noqa: E402


def timeit(fn, s, iters=5):
    ts = []
    for i in range(iters + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def main():
    S, n = 17_301_504, 53
    s = torch.cuda.Stream()
    dst = torch.empty(n * S, dtype=torch.uint8, device="cuda")
    out = {}
    for wc in (False, True):
        h = HostTier(n * S, write_combined=wc)
        sp = F.ptrs_tensor([h.device_address(i * S) for i in range(n)], "cuda")
        dp = F.ptrs_tensor([dst.data_ptr() + i * S for i in range(n)], "cuda")
        sz = F.ptrs_tensor([S] * n, "cuda")
        hs = np.array([h.host_address(i * S) for i in range(n)], dtype=np.uint64)
        hd = np.array([dst.data_ptr() + i * S for i in range(n)], dtype=np.uint64)
        hz = np.full(n, S, dtype=np.uint64)
        r = {}
        for eng in ("ldg", "tma"):
            for mc in (0, 32):
                dt = timeit(lambda: F.batch_copy(sp, dp, sz, engine=eng, max_ctas=mc, stream=s.cuda_stream), s)
                r[f"kernel_{eng}_ctas{mc}_GBps"] = n * S / dt / 1e9
        dt = timeit(lambda: F.ce_batch_copy(hs, hd, hz, batched=True, stream=s.cuda_stream), s)
        r["copy_engine_GBps"] = n * S / dt / 1e9
        page, npg = 65536, 1024
        pp = F.ptrs_tensor([h.device_address(int(p) * page) for p in np.random.default_rng(0).permutation(npg * 4)[:npg]], "cuda")
        dt = timeit(lambda: F.kv_gather(pp, page, dst=dst, stream=s.cuda_stream), s)
        r["kv_1024x64KiB_GBps"] = npg * page / dt / 1e9
        out["write_combined" if wc else "default"] = r
        h.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
