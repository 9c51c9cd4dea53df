"""Device -> pinned host writes (KV evict direction): the SM kernel's
posted stores vs the copy engine, one 16 MiB run x 56 and 1,024 x 64 KiB
pages.  Prints JSON GB/s."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import _native as N  # noqa: E402
from paper_2602_00328_b200.pool import HostTier  # noqa: E402

out = {}
for name, size, n in (("runs_16MiB", 16 << 20, 56), ("pages_64KiB", 65536, 1024), ("expert_17MB", 17_301_504, 53)):
    host = HostTier(size * n)
    dev = torch.empty(size * n, dtype=torch.uint8, device="cuda")
    src = np.array([dev.data_ptr() + i * size for i in range(n)], dtype=np.uint64)
    dst = np.array([host.device_address(i * size) for i in range(n)], dtype=np.uint64)
    sz = np.full(n, size, dtype=np.uint64)
    s = torch.cuda.Stream()
    for eng in ("ldg", "ldg16", "ce"):
        ts = []
        for i in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            N.call("hv_swap_blocks_batch", src.ctypes.data, dst.ctypes.data, sz.ctypes.data, n, N.ENGINES[eng], 0,
                   s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1) * 1e-3)
        out[f"{name}_{eng}_GBps"] = size * n / float(np.median(ts)) / 1e9
    host.close()
print(json.dumps(out, indent=1))
