"""K2 chunk order: linear vs interleaved (HV_ENGINE_FLAG_INTERLEAVE) on the
sources one GPU has (local HBM, pinned host).  One stage of the bench
workload: 53 Qwen experts of 17,301,504 B.  Prints one JSON object (GB/s,
median of 10 launches, L2 flushed between launches)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import fetch as F  # noqa: E402
from paper_2602_00328_b200.pool import HostTier  # noqa: E402


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    S, n = 17_301_504, 53
    dst = torch.empty(n * S, dtype=torch.uint8, device="cuda")
    hbm = torch.empty(n * S, dtype=torch.uint8, device="cuda")
    host = HostTier(n * S)
    dp = F.ptrs_tensor([dst.data_ptr() + i * S for i in range(n)], "cuda")
    sz = F.ptrs_tensor([S] * n, "cuda")
    srcs = {"hbm": F.ptrs_tensor([hbm.data_ptr() + i * S for i in range(n)], "cuda"),
            "host": F.ptrs_tensor([host.device_address(i * S) for i in range(n)], "cuda")}
    out = {}
    s = torch.cuda.current_stream()
    for src_name, sp in srcs.items():
        for eng in ("ldg", "ldg16", "tma"):
            for il in ("", "+il"):
                for grid in (0, 296, 148):
                    ts = []
                    for it in range(13):
                        flush.add_(1)
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(s)
                        F.batch_copy(sp, dp, sz, engine=eng + il, max_ctas=grid)
                        b.record(s)
                        b.synchronize()
                        if it >= 3:
                            ts.append(a.elapsed_time(b) * 1e-3)
                    out[f"{src_name}/{eng}{il}/grid{grid}"] = n * S / float(np.median(ts)) / 1e9
    print(json.dumps(out, indent=1))
    host.close()


if __name__ == "__main__":
    main()
