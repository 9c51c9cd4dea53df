"""Pinned host -> device copy-engine rate with the copies of one stage split
over 1, 2 or 4 streams (cudaMemcpyAsync per object, 53 x 17.3 MB, the Qwen
stage the N=1 bench fetches): does a second DMA engine add PCIe throughput?
Prints JSON: GB/s per stream count, best of 5."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200.pool import HostTier  # noqa: E402


def main():
    S, n = 17_301_504, 53
    host = HostTier(n * S)
    src = torch.from_numpy(host.view())
    dst = torch.empty(n * S, dtype=torch.uint8, device="cuda")
    out = {}
    for k in (1, 2, 3, 4):
        streams = [torch.cuda.Stream() for _ in range(k)]
        best = 0.0
        for _ in range(6):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for st in streams:
                st.wait_event(e0)
            for i in range(n):
                with torch.cuda.stream(streams[i % k]):
                    dst[i * S:(i + 1) * S].copy_(src[i * S:(i + 1) * S], non_blocking=True)
            for st in streams:
                torch.cuda.current_stream().wait_stream(st)
            e1.record()
            e1.synchronize()
            best = max(best, n * S / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out[f"streams{k}"] = best
    host.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
