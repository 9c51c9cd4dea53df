"""Per-fetch content check (hv_check_digests_batch) alone and beside a
concurrent fetch on another stream (copy engine from the host tier, or the
K2 kernel), one Qwen stage (53 x 17.3 MB).  Prints JSON: ms per check."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import _native as N  # noqa: E402
from paper_2602_00328_b200.pool import HostTier  # noqa: E402

S, n = 17_301_504, 53
dev = "cuda:0"
host = HostTier(n * S)
a = torch.zeros(n * S, dtype=torch.uint8, device=dev)
b = torch.empty(n * S, dtype=torch.uint8, device=dev)
pa = np.array([a.data_ptr() + i * S for i in range(n)], dtype=np.uint64)
pb = np.array([b.data_ptr() + i * S for i in range(n)], dtype=np.uint64)
ph = np.array([host.device_address(i * S) for i in range(n)], dtype=np.uint64)
sz = np.full(n, S, dtype=np.uint64)
exp = np.zeros(n, dtype=np.uint64)
scratch = torch.zeros(n, dtype=torch.int64, device=dev)
flags = torch.zeros(n, dtype=torch.uint8, device=dev)
err = torch.zeros(1, dtype=torch.int64, device=dev)
cs, fs = torch.cuda.Stream(), torch.cuda.Stream()


def check():
    N.call("hv_check_digests_batch", pa.ctypes.data, sz.ctypes.data, exp.ctypes.data, n, scratch.data_ptr(),
           flags.data_ptr(), err.data_ptr(), cs.cuda_stream)


def timed_check(bg=None, reps=5):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if bg is not None:
            bg()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        check()
        e1.record(cs)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    return float(np.median(out))


res = {"alone_ms": timed_check()}
for eng in ("ce", "ldg"):
    def bg(eng=eng):
        N.call("hv_swap_blocks_batch", ph.ctypes.data, pb.ctypes.data, sz.ctypes.data, n, N.ENGINES[eng], 0,
               fs.cuda_stream)
    res[f"beside_host_fetch_{eng}_ms"] = timed_check(bg)
print(json.dumps(res, indent=1))
host.close()
