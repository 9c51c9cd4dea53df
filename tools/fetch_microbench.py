"""Fetch-engine microbenchmark on one GPU (sources: local HBM slots, pinned host).

Prints one JSON object.  Used to pick engines/grid sizes; the contract bench is
bench.py.  Times each iteration with CUDA events on the launching stream,
flushing L2 between iterations (256 MiB write).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import fetch as F  # noqa: E402
from paper_2602_00328_b200.pool import HostTier, PeerPool  # noqa: E402


def u64(x):
    return torch.tensor(np.asarray(x, dtype=np.uint64).view(np.int64), device="cuda")


FLUSH = None


def flush():
    FLUSH.add_(1)


def timeit(fn, iters=10, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(iters):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts)), float(np.min(ts))


def main():
    global FLUSH
    torch.cuda.set_device(0)
    FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {"device": torch.cuda.get_device_name(0)}
    page, npages, nslots = 65536, 1024, 4096
    slots_dev = torch.empty(nslots * page, dtype=torch.uint8, device="cuda")
    host = HostTier(nslots * page)
    F.fill_content(u64([slots_dev.data_ptr() + i * page for i in range(nslots)]), u64([page] * nslots),
                   list(range(1, nslots + 1)))
    F.fill_content(u64([host.device_address(i * page) for i in range(nslots)]), u64([page] * nslots),
                   list(range(1, nslots + 1)))
    torch.cuda.synchronize()
    perm = np.random.default_rng(1).permutation(nslots)[:npages]
    dst = torch.empty(npages * page, dtype=torch.uint8, device="cuda")
    nb = npages * page
    res = {}
    for src_name, base in (("hbm", slots_dev.data_ptr()), ("host", host.device_address())):
        sp = u64([base + int(p) * page for p in perm])
        for eng in ("ldg", "ldg256", "ldg16", "tma"):
            for mc in (0, 16, 32, 64):
                med, mn = timeit(lambda: F.kv_gather(sp, page, dst=dst, engine=eng, max_ctas=mc))
                res[f"kv_{src_name}_{eng}_ctas{mc}"] = {"us": med * 1e6, "GBps": nb / med / 1e9}
        hs = np.array([(slots_dev.data_ptr() if src_name == "hbm" else host.host_address()) + int(p) * page
                       for p in perm], dtype=np.uint64)
        hd = np.array([dst.data_ptr() + i * page for i in range(npages)], dtype=np.uint64)
        hz = np.full(npages, page, dtype=np.uint64)
        for bt in (0, 1):
            med, mn = timeit(lambda: F.ce_batch_copy(hs, hd, hz, batched=bool(bt)))
            res[f"kv_{src_name}_ce{'batch' if bt else 'loop'}"] = {"us": med * 1e6, "GBps": nb / med / 1e9}
    out["kv_config1_1024x64KiB"] = res
    # experts
    esz, ne = 17_301_504, 53
    edev = torch.empty(ne * esz, dtype=torch.uint8, device="cuda")
    ehost = HostTier(ne * esz)
    edst = torch.empty(ne * esz, dtype=torch.uint8, device="cuda")
    res = {}
    for src_name, base, hbase in (("hbm", edev.data_ptr(), edev.data_ptr()),
                                  ("host", ehost.device_address(), ehost.host_address())):
        sp = u64([base + i * esz for i in range(ne)])
        dp = u64([edst.data_ptr() + i * esz for i in range(ne)])
        sz = u64([esz] * ne)
        for eng in ("ldg", "ldg256", "ldg16", "tma"):
            for mc in (0, 16, 32, 64):
                med, mn = timeit(lambda: F.batch_copy(sp, dp, sz, engine=eng, max_ctas=mc), iters=5)
                res[f"exp_{src_name}_{eng}_ctas{mc}"] = {"ms": med * 1e3, "GBps": ne * esz / med / 1e9}
        hs = np.array([hbase + i * esz for i in range(ne)], dtype=np.uint64)
        hd = np.array([edst.data_ptr() + i * esz for i in range(ne)], dtype=np.uint64)
        hz = np.full(ne, esz, dtype=np.uint64)
        for bt in (0, 1):
            med, mn = timeit(lambda: F.ce_batch_copy(hs, hd, hz, batched=bool(bt)), iters=5)
            res[f"exp_{src_name}_ce{'batch' if bt else 'loop'}"] = {"ms": med * 1e3, "GBps": ne * esz / med / 1e9}
        # single-expert latency
        for eng in ("ldg", "ldg256", "ldg16", "tma"):
            med, mn = timeit(lambda: F.batch_copy(sp[:1], dp[:1], sz[:1], engine=eng), iters=20)
            res[f"lat1_{src_name}_{eng}_us"] = med * 1e6
        med, mn = timeit(lambda: F.ce_batch_copy(hs[:1], hd[:1], hz[:1], batched=False), iters=20)
        res[f"lat1_{src_name}_ce_us"] = med * 1e6
        if src_name == "host":  # kernel + copy engine concurrently on two streams
            s_ce = torch.cuda.Stream()
            for f in (0.15, 0.3, 0.5, 0.7):
                k = int(round(ne * f))

                def hybrid():
                    cur = torch.cuda.current_stream()
                    s_ce.wait_stream(cur)
                    F.ce_batch_copy(hs[:k], hd[:k], hz[:k], batched=True, stream=s_ce)
                    F.batch_copy(sp[k:], dp[k:], sz[k:], engine="ldg")
                    cur.wait_stream(s_ce)

                med, mn = timeit(hybrid, iters=5)
                res[f"exp_host_hybrid_ce{f}"] = {"ms": med * 1e3, "GBps": ne * esz / med / 1e9}
    out["experts_qwen_53x17.3MB"] = res
    # raw copy peak for reference
    a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    med, mn = timeit(lambda: b.copy_(a), iters=5)
    out["torch_copy_1GiB_GBps_rw"] = 2 * (1 << 30) / med / 1e9
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
