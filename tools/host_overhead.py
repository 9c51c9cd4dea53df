"""Host-side cost of the fetch entry points and the fixed latency of small
fetches (one GPU).  Prints JSON."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import fetch as F  # noqa: E402
from paper_2602_00328_b200.moe import QWEN15_MOE_A27B, ExpertFetcher, ExpertResidency, ExpertStore  # noqa: E402
from paper_2602_00328_b200.system import HarvestSystem  # noqa: E402


def gpu_time(fn, stream, iters=20):
    ts = []
    for i in range(iters + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def main():
    out = {}
    dev = 0
    s = torch.cuda.Stream()
    src = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    dst = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    for nb in (4096, 65536, 1 << 20):
        hs = np.array([src.data_ptr()], dtype=np.uint64)
        hd = np.array([dst.data_ptr()], dtype=np.uint64)
        hz = np.array([nb], dtype=np.uint64)
        sp, dp, sz = (F.ptrs_tensor(x, "cuda") for x in (hs, hd, hz))
        out[f"{nb}B"] = {
            "batch_copy_dev_arrays_us": gpu_time(lambda: F.batch_copy(sp, dp, sz, stream=s.cuda_stream), s),
            "swap_blocks_batch_host_arrays_us": gpu_time(lambda: F.swap_blocks_batch(hs, hd, hz, stream=s.cuda_stream), s),
            "kv_gather_1page_us": gpu_time(lambda: F.kv_gather(sp, nb, dst=dst, stream=s.cuda_stream), s),
            "copy_engine_us": gpu_time(lambda: F.ce_batch_copy(hs, hd, hz, batched=False, stream=s.cuda_stream), s),
            "torch_copy_us": gpu_time(lambda: dst[:nb].copy_(src[:nb]), torch.cuda.current_stream()),
        }
    # ExpertFetcher.issue_fetches host cost per call (53 experts, host tier)
    # 4 KiB "experts": GPU time is negligible, so the host time is the overhead
    m = QWEN15_MOE_A27B
    m = type(m)(m.name, 2, m.num_experts, m.top_k, 4096, hidden=m.hidden, intermediate=m.intermediate)
    sysm = HarvestSystem(dev, host_bytes=2 * m.num_experts * m.expert_size, local_bytes=1, log_transfers=False)
    small = m
    store = ExpertStore(small, sysm.host_id, sysm.host)
    fetcher = ExpertFetcher(sysm.runtime, small, ExpertResidency(small), store)
    stage = torch.empty(m.num_experts * m.expert_size, dtype=torch.uint8, device="cuda")
    ptrs = np.array([stage.data_ptr() + i * m.expert_size for i in range(m.num_experts)], dtype=np.uint64)
    ex = np.arange(0, 53)
    for _ in range(3):
        fetcher.issue_fetches(0, ex, ptrs[:53])
    sysm.loop.run()
    t0 = time.perf_counter()
    n = 50
    for i in range(n):
        fetcher.issue_fetches(i % 2, ex, ptrs[:53])
    host_us = (time.perf_counter() - t0) / n * 1e6
    sysm.loop.run()
    out["issue_fetches_host_us_per_call_53_experts"] = host_us
    import cProfile
    import io
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for i in range(n):
        fetcher.issue_fetches(i % 2, ex, ptrs[:53])
    pr.disable()
    sio = io.StringIO()
    pstats.Stats(pr, stream=sio).sort_stats("tottime").print_stats(12)
    out["profile"] = sio.getvalue().splitlines()[:40]
    sysm.loop.run()
    sysm.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
