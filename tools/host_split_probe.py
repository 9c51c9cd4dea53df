"""Host tier (pinned, PCIe): K2 alone, the copy engine alone, and both at once
on disjoint shares of one Qwen stage (53 experts x 17.3 MB), on two streams.
Prints JSON: GB/s of the whole stage for each split."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import fetch as F  # noqa: E402
from paper_2602_00328_b200.pool import HostTier  # noqa: E402


def main():
    S, n = 17_301_504, 53
    host = HostTier(n * S)
    dst = torch.empty(n * S, dtype=torch.uint8, device="cuda")
    sk, sc = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for k_share in (1.0, 0.0, 0.75, 0.5, 0.25, 0.1):
        nk = int(round(n * k_share))
        kp = F.ptrs_tensor([host.device_address(i * S) for i in range(nk)], "cuda")
        kd = F.ptrs_tensor([dst.data_ptr() + i * S for i in range(nk)], "cuda")
        ks = F.ptrs_tensor([S] * nk, "cuda")
        cs = np.array([host.host_address(i * S) for i in range(nk, n)], dtype=np.uint64)
        cd = np.array([dst.data_ptr() + i * S for i in range(nk, n)], dtype=np.uint64)
        cz = np.full(n - nk, S, dtype=np.uint64)

        def run():
            start = torch.cuda.Event()
            start.record()
            sk.wait_event(start)
            sc.wait_event(start)
            if nk:
                F.batch_copy(kp, kd, ks, stream=sk.cuda_stream)
            if n - nk:
                F.ce_batch_copy(cs, cd, cz, batched=True, stream=sc.cuda_stream)
            torch.cuda.current_stream().wait_stream(sk)
            torch.cuda.current_stream().wait_stream(sc)

        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        out[f"kernel_share_{k_share:.2f}"] = {"ms": ms, "GBps": n * S / (ms * 1e-3) / 1e9}
    host.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
