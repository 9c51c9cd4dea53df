"""K1 block-table form vs per-page pointer form on one GPU (local HBM).

A config-4-shaped reload slice: n_blocks blocks x 32 layers x 64 KiB pages
from peer-slab-like [layer][slot] slabs into a [layer][block] cache.  The
same pages are moved by hv_kv_gather (one pointer pair per page, layer-major)
and by hv_kv_gather_blocks (one base/stride pair per block).  Prints one JSON
object with the median kernel time and algorithmic GB/s per engine.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200 import fetch as F  # noqa: E402


def u64(x):
    return torch.tensor(np.asarray(x, dtype=np.uint64).view(np.int64), device="cuda")


def timeit(fn, flush, iters=10, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(iters):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    page, L, nb, slab_blocks = 65536, 32, int(os.environ.get("KV_PROBE_BLOCKS", "2048")), 256
    nslabs = nb // slab_blocks
    slabs = [torch.empty(L * slab_blocks * page, dtype=torch.uint8, device="cuda") for _ in range(nslabs)]
    cache = torch.empty(L * nb * page, dtype=torch.uint8, device="cuda")
    for s in slabs:
        s.random_(0, 255)
    rng = np.random.default_rng(0)
    order = rng.permutation(nb)  # block i lives at slab/slot order[i]
    sb = np.array([slabs[o // slab_blocks].data_ptr() + (o % slab_blocks) * page for o in order], dtype=np.uint64)
    ss = np.full(nb, slab_blocks * page, dtype=np.uint64)
    db = np.array([cache.data_ptr() + i * page for i in range(nb)], dtype=np.uint64)
    ds = np.full(nb, nb * page, dtype=np.uint64)
    layers = np.arange(L, dtype=np.uint64)[:, None]
    sp = (sb[None, :] + layers * ss[None, :]).reshape(-1)
    dp = (db[None, :] + layers * ds[None, :]).reshape(-1)
    t_sb, t_ss, t_db, t_ds, t_sp, t_dp = (u64(x) for x in (sb, ss, db, ds, sp, dp))
    nbytes = nb * L * page
    out = {"device": torch.cuda.get_device_name(0), "blocks": nb, "layers": L, "page_bytes": page,
           "bytes": nbytes, "engines": {}}
    for eng in ("ldg", "ldg256", "ldg16", "tma"):
        r = {}
        for grid in (0, 296, 148):
            t_pages = timeit(lambda: F.kv_gather(t_sp, page, dst_page_ptrs=t_dp, engine=eng, max_ctas=grid), flush)
            t_blocks = timeit(lambda: F.kv_gather_blocks(t_sb, t_ss, t_db, t_ds, L, page, engine=eng,
                                                         max_ctas=grid), flush)
            r[f"grid{grid}"] = {"pages_ms": t_pages * 1e3, "blocks_ms": t_blocks * 1e3,
                                "pages_GBps": nbytes / t_pages / 1e9, "blocks_GBps": nbytes / t_blocks / 1e9}
        out["engines"][eng] = r
    # parity of the two forms on this layout
    cache.zero_()
    F.kv_gather_blocks(t_sb, t_ss, t_db, t_ds, L, page)
    ref = torch.empty_like(cache)
    F.kv_gather(t_sp, page, dst_page_ptrs=u64((dp - np.uint64(cache.data_ptr()) + np.uint64(ref.data_ptr()))))
    torch.cuda.synchronize()
    out["forms_identical"] = bool(torch.equal(cache, ref))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
