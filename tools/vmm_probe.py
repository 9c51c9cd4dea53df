"""Cost of VMM commit/decommit (cuMemCreate+Map+SetAccess / Unmap+Release)
per chunk size, for 1 GiB of harvested segments.  Prints JSON."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00328_b200.pool import PeerPool  # noqa: E402


def main():
    out = {}
    seg = 17_301_504
    n = 60
    for chunk in (2 << 20, 8 << 20, 32 << 20, 64 << 20):
        p = PeerPool(0, n * seg + (64 << 20), readers=[0], chunk_bytes=chunk)
        t0 = time.perf_counter()
        for i in range(n):
            p.commit(i * seg, seg)
        t1 = time.perf_counter()
        for i in range(n):
            p.decommit(i * seg, seg)
        t2 = time.perf_counter()
        out[f"chunk_{chunk >> 20}MiB"] = {"commit_ms_per_expert": (t1 - t0) / n * 1e3,
                                          "decommit_ms_per_expert": (t2 - t1) / n * 1e3}
        p.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
